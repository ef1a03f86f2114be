// Prefill causal flash attention on the 5th-generation tensor cores (sm_100a,
// bf16): a T-token chunk at positions [p0, p0+T) attends cache rows [0, p0+T)
// (blockwise online softmax math.hpp:56-101, partition-invariant
// SPEC.md:312).
//
// One CTA per (128-query tile, head, sequence), warp-specialized:
//   warp 0      TMA producer: the Q tile once, then 128-key K and V tiles
//               (SWIZZLE_128B boxes of 64 dims x 128 rows) into a 2-stage ring;
//   warp 1      MMA issuer (one thread): S = Q.K^T into one of two TMEM score
//               buffers (M = 128 queries, N = 128 keys, K = d_head), then
//               O_j = P.V into a TMEM tile (A = P from shared memory, K-major;
//               B = V straight from the cache layout, MN-major);
//   warps 2..5  softmax, one query row per thread (TMEM lane = row): row max
//               over the S row, exp2, P (bf16) into shared memory in the MMA's
//               K-major SW128 image, and O += O_j with the running-max rescale
//               in registers. S of tile j+1 is computed while tile j's softmax
//               runs.
#include <cuda.h>
#include <math_constants.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace fsvd::k {
namespace {

constexpr int kAQ = 128, kAK = 128;    // queries per CTA, keys per tile
constexpr int kAThreads = 320;         // producer, MMA, 8 softmax warps (two per TMEM lane group)
constexpr int kBox = kAK * 128;        // one 64-dim x 128-row SW128 box: 16 KiB

struct AttnTcArgs {
    CUtensorMap qmap, kmap, vmap;  // {d, rows} bf16, box {64, 128}, SWIZZLE_128B
    AttnPrefillArgs a;
    long long kv_row_b, kv_row_h;  // cache row of (b, h, pos) = b kv_row_b + h kv_row_h + pos
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "W_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n"
        "}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            su32(dst)),
        "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// SW128 shared-memory descriptors (8-row x 128 B atoms at 1024 B).
// K-major: rows = M/N index, 64 K-elements per 128 B row.
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
    return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
// MN-major: rows = K index (8-row atoms at SBO = 1024 B), 64 N-elements per
// 128 B row, the next 64 N-elements at LBO = one 16 KiB box.
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {
    return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(kBox >> 4) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16 instruction descriptor: D f32, A/B bf16, A K-major, B K- or MN-major
template <int M, int N, bool B_MN>
__device__ __forceinline__ constexpr uint32_t idesc() {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((B_MN ? 1u : 0u) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

template <int DH>
__global__ void __launch_bounds__(kAThreads, 1) attn_tc_kernel(const __grid_constant__ AttnTcArgs A) {
    static_assert(DH == 64 || DH == 128, "d_head");
    constexpr int NB = DH / 64;                 // 64-dim boxes per row tile
    constexpr uint32_t kTile = NB * kBox;       // Q / K / V tile bytes
    constexpr uint32_t kOcol = 256;             // TMEM: S buffers at columns 0 / 128, O_j at 256
    const AttnPrefillArgs& a = A.a;
    extern __shared__ __align__(1024) uint8_t sraw[];
    // (no alignment slack: Q, 2 x K, 2 x V and 2 x P fill 224 KiB at d_head 128; the
    // dynamic shared window starts on a 1 KiB boundary -- checked below)
    uint8_t* sm = sraw;
    uint8_t* Qs = sm;
    uint8_t* Ks = Qs + kTile;           // [2] stages
    uint8_t* Vs = Ks + 2 * kTile;       // [2]
    uint8_t* Ps = Vs + 2 * kTile;       // [2] 128 queries x 128 keys bf16, K-major SW128 (2 boxes each)
    uint64_t* bars = reinterpret_cast<uint64_t*>(Ps + 4 * kBox);
    uint64_t *q_full = bars, *kv_full = bars + 1, *kv_empty = bars + 3, *s_full = bars + 5, *s_empty = bars + 7,
             *p_full = bars + 9, *pv_done = bars + 10;  // pv_done[2]: P.V of the tiles using P buffer 0 / 1
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 12);
    float* xch = reinterpret_cast<float*>(bars + 16);  // [2 parities][2 halves][128] row exchange
    if ((su32(sraw) & 1023u) != 0) __trap();

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // q, the cache rows and the length register
    const int qt = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, b = blockIdx.z;  // heaviest causal tiles first
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q0 = qt * kAQ;
    const int p0 = a.p0_dev ? *a.p0_dev : a.p0;
    const int last_q = min(a.T, q0 + kAQ) - 1;
    const int kend = p0 + last_q + 1;  // keys this tile needs
    const int ntiles = (kend + kAK - 1) / kAK;

    if (threadIdx.x == 0) {
        bar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            bar_init(&kv_full[i], 1);
            bar_init(&kv_empty[i], 1);
            bar_init(&s_full[i], 1);
            bar_init(&s_empty[i], 256);
        }
        bar_init(p_full, 256);
        bar_init(&pv_done[0], 1);
        bar_init(&pv_done[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            bar_expect(q_full, kTile);
            for (int i = 0; i < NB; ++i) tma2d(Qs + i * kBox, &A.qmap, q_full, h * DH + 64 * i, b * a.T + q0);
            const int row0 = static_cast<int>(b * A.kv_row_b + h * A.kv_row_h);
            for (int j = 0; j < ntiles; ++j) {
                const int st = j & 1;
                bar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
                bar_expect(&kv_full[st], 2 * kTile);
                for (int i = 0; i < NB; ++i) {
                    tma2d(Ks + st * kTile + i * kBox, &A.kmap, &kv_full[st], 64 * i, row0 + j * kAK);
                    tma2d(Vs + st * kTile + i * kBox, &A.vmap, &kv_full[st], 64 * i, row0 + j * kAK);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id_s = idesc<kAQ, kAK, false>();  // S[q][key] = Q . K^T, K = d
            constexpr uint32_t id_o = idesc<kAQ, DH, true>();    // O[q][d] = P . V,  K = keys
            bar_wait(q_full, 0);
            auto issue_s = [&](int j) {
                const int st = j & 1;
                bar_wait(&kv_full[st], (j >> 1) & 1);
                bar_wait(&s_empty[st], ((j >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t qa = su32(Qs), ka = su32(Ks + st * kTile);
#pragma unroll
                for (int k = 0; k < DH / 16; ++k)  // 16 dims per MMA: +32 B inside a 64-dim box
                    mma(tmem + st * kAK, desc_k(qa + (k >> 2) * kBox) + 2 * (k & 3),
                        desc_k(ka + (k >> 2) * kBox) + 2 * (k & 3), id_s, k > 0);
                commit(&s_full[st]);
            };
            issue_s(0);
            for (int j = 0; j < ntiles; ++j) {
                const int st = j & 1;
                if (j + 1 < ntiles) issue_s(j + 1);
                bar_wait(p_full, j & 1);  // P_j written (and O rescaled, if the running max moved)
                fence_after();
                const uint32_t pa = su32(Ps + (j & 1) * 2 * kBox), va = su32(Vs + st * kTile);
#pragma unroll
                for (int kk = 0; kk < kAK / 16; ++kk)  // 16 keys per MMA: P +32 B, V +16 rows (2 KiB)
                    mma(tmem + kOcol, desc_k(pa + (kk >> 2) * kBox) + 2 * (kk & 3), desc_mn(va + kk * 2048), id_o,
                        (j > 0 || kk > 0) ? 1u : 0u);  // O accumulates in TMEM over the key tiles
                commit(&pv_done[j & 1]);
                commit(&kv_empty[st]);
            }
        }
    } else {
        // softmax: query row r = TMEM lane; two threads per row (warps 2-5 and 6-9 see
        // the same TMEM lanes), half hf owns keys [64 hf, 64 hf + 64) of every tile and
        // output columns [hf DH/2, hf DH/2 + DH/2). Each S row is read from TMEM once
        // (into registers); O accumulates in TMEM (P.V with accumulate) and is rescaled
        // there only when the running max grows by more than kTau (log2 units) -- exact,
        // since P and the row sum use the same reference max. P is double-buffered, so
        // writing P_j waits for P.V of tile j - 2, not j - 1. The row max is exchanged
        // through shared memory, the row sums only at the end.
        constexpr int DH2 = DH / 2;
        constexpr float kTau = 8.0f;
        const int hf = (warp - 2) >> 2;
        const int r = (warp & 3) * 32 + lane;
        const int t = q0 + r, qpos = p0 + t;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        const uint32_t ocol = lane_base + kOcol + hf * DH2;
        const float sl2 = a.scale * 1.4426950408889634f;  // scores in log2 units
        float m = -CUDART_INF_F, l = 0.f;
        // P.V of tile i has completed: completion (i >> 1) of pv_done[i & 1] (parity (i >> 1) & 1)
        auto wait_pv = [&](int i) { bar_wait(&pv_done[i & 1], (i >> 1) & 1); };
        for (int j = 0; j < ntiles; ++j) {
            const int st = j & 1, k0 = j * kAK + hf * 64;
            const uint32_t scol = lane_base + st * kAK + hf * 64;
            uint8_t* prow = Ps + (j & 1) * 2 * kBox + hf * kBox + r * 128;  // P buffer j & 1, box hf
            bar_wait(&s_full[st], (j >> 1) & 1);
            fence_after();
            float sv[64];
            {
                float v[32];
                tmem_ld32(scol, v);
#pragma unroll
                for (int i = 0; i < 32; ++i) sv[i] = v[i];
                tmem_ld32(scol + 32, v);
#pragma unroll
                for (int i = 0; i < 32; ++i) sv[32 + i] = v[i];
            }
            fence_before();
            bar_arrive(&s_empty[st]);  // the S buffer is free for tile j + 2
            float mx = -CUDART_INF_F;
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                sv[i] = k0 + i <= qpos ? sv[i] * sl2 : -CUDART_INF_F;
                mx = fmaxf(mx, sv[i]);
            }
            xch[((j & 1) * 2 + hf) * kAQ + r] = mx;
            asm volatile("bar.sync 1, 256;" ::: "memory");
            mx = fmaxf(mx, xch[((j & 1) * 2 + (hf ^ 1)) * kAQ + r]);
            if (mx != -CUDART_INF_F && (m == -CUDART_INF_F || mx > m + kTau)) {
                const float f = m == -CUDART_INF_F ? 0.f : exp2f(m - mx);
                if (j > 0 && m != -CUDART_INF_F) {  // O *= f in TMEM once P.V of tile j - 1 is done (rare)
                    wait_pv(j - 1);
                    fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < DH2; c0 += 32) {
                        float v[32];
                        tmem_ld32(ocol + c0, v);
                        uint32_t w[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(v[i] * f);
                        asm volatile(
                            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
                                ocol + c0),
                            "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
                            "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
                            "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]),
                            "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]),
                            "r"(w[29]), "r"(w[30]), "r"(w[31])
                            : "memory");
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                }
                l *= f;
                m = mx;
            }
            if (j >= 2) wait_pv(j - 2);  // P buffer j & 1 was read by P.V of tile j - 2
            // P = exp2(s - m) in bf16 into the K-major SW128 image (row r of box hf,
            // 16-B chunk c at c ^ (r & 7))
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 32) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    const float s0 = m == -CUDART_INF_F ? 0.f : exp2f(sv[c0 + i] - m);
                    const float s1 = m == -CUDART_INF_F ? 0.f : exp2f(sv[c0 + i + 1] - m);
                    l += s0 + s1;
                    pk[i >> 1] = pack2(s0, s1);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int chunk = (c0 >> 3) + u;
                    *reinterpret_cast<uint4*>(prow + ((chunk ^ (r & 7)) << 4)) =
                        make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
                }
            }
            if (j * kAK + kAK > kend && hf < NB) {
                // last tile: V rows past the history are not this sequence's (stale or
                // never written) -- zero them (box hf) so 0 * garbage cannot reach O
                if (j * kAK + r >= kend) {
                    uint8_t* vrow = Vs + st * kTile + hf * kBox + r * 128;
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        *reinterpret_cast<uint4*>(vrow + c * 16) = make_uint4(0u, 0u, 0u, 0u);
                }
            }
            fence_before();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P / V stores -> the tensor core
            bar_arrive(p_full);
        }
        wait_pv(ntiles - 1);
        fence_after();
        // row sum = both halves' partial sums (same reference max); the exchange slot of
        // parity ntiles & 1 was last read before the final iteration's barrier
        xch[((ntiles & 1) * 2 + hf) * kAQ + r] = l;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        l += xch[((ntiles & 1) * 2 + (hf ^ 1)) * kAQ + r];
        const float inv = 1.f / l;
        __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.out) + static_cast<long long>(b * a.T + t) * a.out_ld +
                              h * DH + hf * DH2;
#pragma unroll
        for (int c0 = 0; c0 < DH2; c0 += 32) {
            float v[32];
            tmem_ld32(ocol + c0, v);  // (all lanes: .sync.aligned)
            if (t < a.T) {
#pragma unroll
                for (int e = 0; e < 32; e += 8)
                    *reinterpret_cast<uint4*>(orow + c0 + e) =
                        make_uint4(pack2(v[e] * inv, v[e + 1] * inv), pack2(v[e + 2] * inv, v[e + 3] * inv),
                                   pack2(v[e + 4] * inv, v[e + 5] * inv), pack2(v[e + 6] * inv, v[e + 7] * inv));
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode() {
    static EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeTiled>(p);
    }();
    return fn;
}
void map2d(CUtensorMap* m, const void* base, long long cols, long long rows, long long ld) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("attn_tc: cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

}  // namespace

bool attn_prefill_tcgen05(const AttnPrefillArgs& a, cudaStream_t s) {
    if (std::getenv("FSVD_ATTN_MMA")) return false;
    if (a.d_head != 64 && a.d_head != 128) return false;
    if (a.q_ld % 8 || a.out_ld % 8 || a.cache_hstride % a.d_head || a.cache_bstride % a.d_head) return false;
    if ((reinterpret_cast<uintptr_t>(a.q) | reinterpret_cast<uintptr_t>(a.out)) & 15) return false;
    AttnTcArgs A{};
    A.a = a;
    A.kv_row_b = a.cache_bstride / a.d_head;
    A.kv_row_h = a.cache_hstride / a.d_head;
    const long long kv_rows = a.batch * A.kv_row_b;
    map2d(&A.qmap, a.q, a.q_ld, static_cast<long long>(a.batch) * a.T, a.q_ld);
    map2d(&A.kmap, a.kcache, a.d_head, kv_rows, a.d_head);
    map2d(&A.vmap, a.vcache, a.d_head, kv_rows, a.d_head);
    const int NB = a.d_head / 64;
    const int smem = 5 * NB * kBox + 4 * kBox + 128 + 4 * 128 * 4;  // Q, 2 x K, 2 x V, 2 x P, barriers, row exchange
    dim3 grid((a.T + kAQ - 1) / kAQ, a.n_heads, a.batch);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kAThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = std::getenv("FSVD_NO_PDL") ? 0 : 1;
    if (a.d_head == 128) {
        cudaFuncSetAttribute(attn_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaLaunchKernelEx(&cfg, attn_tc_kernel<128>, A);
    } else {
        cudaFuncSetAttribute(attn_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaLaunchKernelEx(&cfg, attn_tc_kernel<64>, A);
    }
    return true;
}

}  // namespace fsvd::k
