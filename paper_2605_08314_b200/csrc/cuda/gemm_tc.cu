// Prefill GEMM on the 5th-generation tensor cores (sm_100a, bf16 mode):
//
//   Y[t][n] = epi( sum_k X[t][k] * W^T[n][k] )      (SPEC.md:305-313 prefill:
//   P = X.A once for the whole prompt, then P.B with the RoPE / KV-write,
//   residual and SiLU.mul epilogues)
//
// One CTA per 128 x BN output tile, warp-specialized:
//   warp 0      TMA producer: X tile (128 tokens x 64 k, SWIZZLE_128B) via a
//               tensor map (cp.async.bulk.tensor.2d), W^T tile as ONE 4-D
//               tensor-map box {64 el, 16 rows, line, BN/16 tiles} over the
//               device weight layout (layout.h), which already IS the K-major
//               SWIZZLE_128B core-matrix image, so weights land verbatim;
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma
//               (kind::f16, M=128, N=BN, K=16) into a TMEM fp32 accumulator
//               and tcgen05.commit's each stage back to the producer;
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 32 columns per warp, then
//               the fused epilogue straight from registers.
// The dual (up/gate) GEMM runs the two K-loops into two TMEM accumulators and
// applies silu(gate) * up in the epilogue, so up/gate never reach memory.
// CG = 2 runs a CTA pair (tcgen05.mma.cta_group::2, M = 256 over two SMs, each
// CTA holding half of the W tile); K splits of a tile can form one thread-block
// cluster and reduce their fp32 partials through DSMEM before the epilogue
// (A.cred), instead of a workspace round trip and splitk_reduce_kernel.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace fsvd::k {
namespace {

using namespace fsvd::dev;

constexpr int BM = 128, BK = 64;
constexpr int kABytes = BM * 128;  // 16 KiB: 128 rows x 128 B
constexpr int kThreads = 192;

template <int BN, int BMT = 1, int CG = 1>
struct Cfg {
    static constexpr int kBBytes = BN / CG * 128;  // a CTA pair holds half of the W tile in each CTA
    static constexpr int kStageBytes = BMT * kABytes + kBBytes;
    static constexpr int kStages = (200 * 1024) / kStageBytes;
    static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

struct TcArgs {
    CUtensorMap xmap;     // X [rows][x_ld] bf16, box 64 x 128, SWIZZLE_128B
    CUtensorMap wmap[3];  // W^T of each segment as {64 el, 16 rows, lines, tiles}: one TMA per stage copies
                          // line kb of BN/16 tiles verbatim (the layout is already the SW128 image)
    GemmArgs g;
    int seg_tiles[3];  // BN-wide output tiles per segment
    int splits;        // split-K factor (blockIdx.z = split; > 1 only for kGemmStore / kGemmAddF32)
    int cred;          // 1: the splits of a tile form one thread-block cluster and reduce through DSMEM
    int dbg;           // development: bit 0 = skip the MMAs (operand-stream-only timing)
};

// ----------------------------------------------------------------- PTX ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// CTA-pair forms: the destination is this CTA's shared memory, the mbarrier the
// leader CTA's (cta_group::2 lets the completion land in the peer of the pair)
__device__ __forceinline__ void tma_load_4d_cg2(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
        "%5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}
// shared::cluster address of the same object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// completion of the pair's MMAs -> the same mbarrier in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// CTA pair: D[tmem of both CTAs] (+)= A[rows 0-127 in CTA 0, 128-255 in CTA 1] .
// B[half of the N rows in each CTA]^T; issued by the leader CTA only
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
// D[tmem] (+)= A[smem] . B[smem]^T, bf16 in, fp32 accumulate
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
// K-major SWIZZLE_128B shared-memory matrix descriptor (8-row x 128 B atoms
// stacked at 1024 B): start>>4 [0,14), LBO [16,30) (unused for SW128 K-major),
// SBO>>4 [32,46), version 1 [46,48), layout SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
// instruction descriptor, kind::f16: D f32, A/B bf16, both K-major
template <int N, int MM = BM>
__device__ __forceinline__ constexpr uint32_t idesc_bf16() {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(MM >> 4) << 24);
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

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}
// 32 consecutive bf16 outputs (64 B, 16 B aligned) from fp32 values
__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float (&v)[32], int valid) {
    if (valid >= 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            d4[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                               pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (i < valid) dst[i] = __float2bfloat16_rn(v[i]);
    }
}

// RMSNorm fold: 1 / rms of row t from the per-32-column sums of squares of the
// producing residual epilogue (GemmArgs::norm_ss_in), summed in index order
__device__ __forceinline__ float norm_row_scale(const GemmArgs& g, int t) {
    if (!g.norm_ss_in || t >= g.M) return 1.f;
    const float4* p = reinterpret_cast<const float4*>(g.norm_ss_in + static_cast<long long>(t) * g.norm_ss_ld);
    // 8 loads in flight per round, four partial sums, combined in a fixed order
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    const int n4 = g.norm_ss_n / 4;
    for (int j = 0; j < n4; j += 8) {
        float4 q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = j + u < n4 ? __ldg(p + j + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s0 += q[u].x;
            s1 += q[u].y;
            s2 += q[u].z;
            s3 += q[u].w;
        }
    }
    const float ss = (s0 + s1) + (s2 + s3);
    return 1.0f / sqrtf(ss / static_cast<float>(g.norm_d) + g.norm_eps);
}

// -------------------------------------------------------------- kernel ----
// BMT = 128-row M sub-tiles per CTA sharing each W tile (2: a 256 x BN tile in
// two TMEM accumulators -- half the W traffic per FLOP of BMT = 1).
//
// CG = 2: a CTA pair (cluster of 2 on one TPC) computes a (CG*128*BMT) x BN tile
// with tcgen05.mma.cta_group::2 (M = 256): each CTA loads its own 128-row X
// sub-tiles and HALF of the W tile, the leader CTA issues the MMAs for both and
// each CTA's TMEM holds its own rows' accumulators -- half the W bytes per SM
// of CG = 1 at the same per-SM tile and MMA time.
template <int BN, bool DUAL, int BMT, int CG>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc_kernel(const __grid_constant__ TcArgs A) {
    static_assert(!(DUAL && BMT > 1), "the dual GEMM uses the second accumulator for the gate");
    static_assert(CG == 1 || (BN / CG) % 16 == 0, "pair halves of the W tile are whole 16-row core-matrix groups");
    using C = Cfg<BN, BMT, CG>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* tmem_full = empty + C::kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const GemmArgs& g = A.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // output tile -> (segment, n0)
    int tile = blockIdx.y, s = 0;
    if constexpr (!DUAL) {
        while (s + 1 < g.nseg && tile >= A.seg_tiles[s]) {
            tile -= A.seg_tiles[s];
            ++s;
        }
    }
    const GemvSeg& sg = g.seg[s];
    // cluster rank = x + CG z (x: CTA of the pair, z: K split when the splits share a cluster)
    const uint32_t crank = (CG == 2 || A.cred) ? cluster_ctarank() : 0u;
    const uint32_t rank = crank % CG, lead = crank - rank;  // pair rank, the pair leader's cluster rank
    const bool leader = rank == 0;
    // rows of M sub-tile mi held by this CTA: pair base + mi * (CG * 128) + rank * 128
    const int n0 = tile * BN, m0 = (blockIdx.x / CG) * BM * BMT * CG + static_cast<int>(rank) * BM;
    constexpr int kAcc = DUAL ? 2 : 1;
    constexpr uint32_t kAccStride = 256;  // dual: gate accumulator at TMEM column 256
    constexpr uint32_t kCols = (DUAL || BMT > 1) ? 2 * kAccStride : BN;
    constexpr uint32_t kAllocCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&A.xmap) : "memory");
    }
    if (warp == 0) {
        if constexpr (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kAllocCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kAllocCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    if constexpr (CG == 2)
        cluster_sync_all();  // both CTAs' barriers initialised before any TMA / commit crosses the pair
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // K-loop of accumulator j: segment, x column offset, k-blocks
    auto seg_of = [&](int j) -> const GemvSeg& { return DUAL ? g.seg[j] : sg; };
    // fused epilogue of one 32-column chunk of output row t (columns n0 + c0 ..)
    auto emit = [&](int t, int c0, float (&v)[32], float rs) {
        const int n = n0 + c0;
        const int valid = min(32, sg.rows - n);
        if (t >= g.M || valid <= 0) return;
        if constexpr (DUAL) {  // v = silu(gate) * up already
            store_bf16x32(static_cast<__nv_bfloat16*>(g.y) + static_cast<long long>(t) * g.y_ld + sg.y_off + n, v,
                          valid);
        } else if (A.splits > 1 && !A.cred) {  // fp32 partial of this K split (plain store / residual add)
            float* w = g.ws + (static_cast<size_t>(blockIdx.z) * g.M + t) * g.y_ld + sg.y_off + n;
            if (valid == 32 && (reinterpret_cast<uintptr_t>(w) & 15) == 0) {  // whole sectors
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                    __stcs(reinterpret_cast<float4*>(w + i), make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i < valid) w[i] = v[i];
            }
        } else if (g.epi == kGemmStore) {
            if (g.norm_ss_in) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] *= rs;
            }
            store_bf16x32(static_cast<__nv_bfloat16*>(g.y) + static_cast<long long>(t) * g.y_ld + sg.y_off + n, v,
                          valid);
        } else if (g.epi == kGemmAddF32) {
            float* y = static_cast<float*>(g.y) + static_cast<long long>(t) * g.y_ld + sg.y_off + n;
            if (valid == 32 && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {  // whole sectors
                float4 r[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) r[i] = reinterpret_cast<const float4*>(y)[i];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    r[i] = make_float4(r[i].x + v[4 * i], r[i].y + v[4 * i + 1], r[i].z + v[4 * i + 2],
                                       r[i].w + v[4 * i + 3]);
                    reinterpret_cast<float4*>(y)[i] = r[i];
                }
                if (g.norm_xg) {  // the next RMSNorm's operands: x_new * gamma in bf16, sum of squares
                    const float4* gm = reinterpret_cast<const float4*>(g.norm_gamma + sg.y_off + n);
                    float ss = 0.f;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float4 gv = __ldg(gm + i);
                        ss = fmaf(r[i].x, r[i].x, ss);
                        ss = fmaf(r[i].y, r[i].y, ss);
                        ss = fmaf(r[i].z, r[i].z, ss);
                        ss = fmaf(r[i].w, r[i].w, ss);
                        v[4 * i] = r[i].x * gv.x;
                        v[4 * i + 1] = r[i].y * gv.y;
                        v[4 * i + 2] = r[i].z * gv.z;
                        v[4 * i + 3] = r[i].w * gv.w;
                    }
                    store_bf16x32(static_cast<__nv_bfloat16*>(g.norm_xg) + static_cast<long long>(t) * g.norm_xg_ld +
                                      sg.y_off + n,
                                  v, 32);
                    g.norm_ss[static_cast<long long>(t) * g.norm_ss_ld + (sg.y_off + n) / 32] = ss;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i < valid) y[i] += v[i];
            }
        } else {  // kGemmQKV: RoPE (interleaved pairs, math.hpp:30-44) + q store / KV append
            const int b = t / g.T, pos = (g.p0_dev ? *g.p0_dev : g.p0) + t % g.T;
            if (sg.epi != kEpiV) {
                // the 32-column chunk lies inside one head (d_head is a multiple of 32): its 16
                // (cos, sin) pairs are contiguous -- 8 vector loads, no per-pair index math
                const float4* cs = reinterpret_cast<const float4*>(
                    g.rope + static_cast<long long>(pos) * (g.d_head / 2) + ((n % g.d_head) >> 1));
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 c = __ldg(cs + q);
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int i = 4 * q + 2 * u;
                        const float cx = u ? c.z : c.x, cy = u ? c.w : c.y;
                        const float x0 = v[i], x1 = v[i + 1];
                        v[i] = __fsub_rn(__fmul_rn(x0, cx), __fmul_rn(x1, cy));
                        v[i + 1] = __fadd_rn(__fmul_rn(x0, cy), __fmul_rn(x1, cx));
                    }
                }
            }
            if (sg.epi == kEpiRopeQ) {
                store_bf16x32(static_cast<__nv_bfloat16*>(g.y) + static_cast<long long>(t) * g.y_ld + sg.y_off + n,
                              v, valid);
            } else {
                const int h = n / g.d_head, ih = n % g.d_head;
                __nv_bfloat16* c = static_cast<__nv_bfloat16*>(sg.epi == kEpiRopeK ? g.kcache : g.vcache);
                store_bf16x32(c + b * g.cache_bstride + h * g.cache_hstride + static_cast<long long>(pos) * g.d_head +
                                  ih,
                              v, valid);
            }
        }
    };

    // Programmatic dependent launch: this grid may start while the previous
    // kernel drains. Only the weight tiles (constant) are read before
    // griddepcontrol.wait; activations are read and outputs written after it.
    float rs_epi = 1.f;  // epilogue threads: the folded RMSNorm scale of their row (cluster path)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp == 0) {
        if (lane == 0) {
            auto kb_range = [&](int j, int& kb0, int& kb1) {
                const int nk = seg_of(j).layout(2).nlines();
                kb0 = nk * static_cast<int>(blockIdx.z) / A.splits;
                kb1 = nk * (static_cast<int>(blockIdx.z) + 1) / A.splits;
            };
            // development (dbg bit 1): rotate each CTA's k-block order by its N tile
            auto kk = [&](int kb, int kb0, int kb1) {
                if (!(A.dbg & 2)) return kb;
                const int n = kb1 - kb0;
                return kb0 + (kb - kb0 + static_cast<int>(blockIdx.y) * 5) % n;
            };
            const int t0 = n0 / 16 + static_cast<int>(rank) * (BN / CG / 16);  // this CTA's half of the W tile
            // the W box always lands whole (tiles past the end are zero-filled); the
            // leader's full barrier counts the bytes of both CTAs of a pair
            const uint32_t bytes = CG * (BMT * kABytes + static_cast<uint32_t>(BN / CG / 16) * kLineTileBytes);
            auto load_w = [&](int st, const CUtensorMap* wm, int kb) {
                uint8_t* dst = smem + st * C::kStageBytes + BMT * kABytes;
                if constexpr (CG == 2) {
                    if (leader) mbar_expect_tx(&full[st], bytes);
                    tma_load_4d_cg2(dst, wm, mapa_u32(&full[st], lead), 0, 0, kb, t0);
                } else {
                    mbar_expect_tx(&full[st], bytes);
                    tma_load_4d(dst, wm, &full[st], 0, 0, kb, t0);
                }
            };
            auto load_x = [&](int st, int mi, int kcol) {
                uint8_t* dst = smem + st * C::kStageBytes + mi * kABytes;
                if constexpr (CG == 2)
                    tma_load_2d_cg2(dst, &A.xmap, mapa_u32(&full[st], lead), kcol, m0 + mi * BM * CG);
                else
                    tma_load_2d(dst, &A.xmap, &full[st], kcol, m0 + mi * BM);
            };
            // W tiles of the first ring round, ahead of the grid dependency
            int npre = 0;
            for (int j = 0; j < kAcc && npre < C::kStages; ++j) {
                int kb0, kb1;
                kb_range(j, kb0, kb1);
                for (int kb = kb0; kb < kb1 && npre < C::kStages; ++kb, ++npre)
                    load_w(npre, &A.wmap[DUAL ? j : s], kk(kb, kb0, kb1));
            }
            asm volatile("griddepcontrol.wait;" ::: "memory");
            int it = 0;
#pragma unroll 1
            for (int j = 0; j < kAcc; ++j) {
                const GemvSeg& sj = seg_of(j);
                const CUtensorMap* wm = &A.wmap[DUAL ? j : s];
                int kb0, kb1;
                kb_range(j, kb0, kb1);
#pragma unroll 1
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int st = it % C::kStages;
                    const uint32_t ph = (it / C::kStages) & 1;
                    if (it >= npre) {
                        mbar_wait(&empty[st], ph ^ 1);
                        load_w(st, wm, kk(kb, kb0, kb1));
                    }
#pragma unroll
                    for (int mi = 0; mi < BMT; ++mi) load_x(st, mi, sj.x_off + kk(kb, kb0, kb1) * BK);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            constexpr uint32_t idesc = idesc_bf16<BN, BM * CG>();
            int it = 0;
#pragma unroll 1
            for (int j = 0; j < kAcc; ++j) {
                const int nk = seg_of(j).layout(2).nlines();
                const int kb0 = nk * static_cast<int>(blockIdx.z) / A.splits;
                const int kb1 = nk * (static_cast<int>(blockIdx.z) + 1) / A.splits;
                const uint32_t tacc = tmem_base + static_cast<uint32_t>(j) * kAccStride;
#pragma unroll 1
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int st = it % C::kStages;
                    const uint32_t ph = (it / C::kStages) & 1;
                    mbar_wait(&full[st], ph);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + st * C::kStageBytes);
                    const uint32_t sb = sa + BMT * kABytes;
                    const uint64_t db = sw128_desc(sb);
                    if (!(A.dbg & 1)) {
#pragma unroll
                        for (int mi = 0; mi < BMT; ++mi) {
                            const uint64_t da = sw128_desc(sa + mi * kABytes);
#pragma unroll
                            for (int k = 0; k < BK / 16; ++k) {  // +32 B per K=16 step inside the 128 B swizzle atom
                                if constexpr (CG == 2)
                                    tc_mma_pair(tacc + mi * kAccStride, da + 2 * k, db + 2 * k, idesc,
                                                (kb != kb0 || k != 0) ? 1u : 0u);
                                else
                                    tc_mma(tacc + mi * kAccStride, da + 2 * k, db + 2 * k, idesc,
                                           (kb != kb0 || k != 0) ? 1u : 0u);
                            }
                        }
                    }
                    if constexpr (CG == 2)
                        tc_commit_pair(&empty[st], static_cast<uint16_t>(3u << lead));
                    else
                        tc_commit(&empty[st]);
                }
            }
            if constexpr (CG == 2)
                tc_commit_pair(tmem_full, static_cast<uint16_t>(3u << lead));
            else
                tc_commit(tmem_full);
        }
    } else {
        // epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 (= tile rows)
        const int q = warp & 3;
        const int row = q * 32 + lane;
        asm volatile("griddepcontrol.wait;" ::: "memory");
        // folded RMSNorm row scales, read while the mainloop runs
        const float rs_mi[2] = {norm_row_scale(g, m0 + row), BMT > 1 ? norm_row_scale(g, m0 + BM * CG + row) : 1.f};
        rs_epi = rs_mi[0];
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        if (!DUAL && A.cred) {
            // cluster split-K: this split's fp32 partial -> own smem as [column][row]
            // (the ring is idle: every MMA that read it has completed)
            float* red = reinterpret_cast<float*>(smem);
            const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                float v[32];
                tmem_ld32(lane_addr + c0, v);
#pragma unroll
                for (int i = 0; i < 32; ++i) red[(c0 + i) * BM + row] = v[i];
            }
        } else {
#pragma unroll 1
            for (int mi = 0; mi < BMT; ++mi) {
                const int t = m0 + mi * BM * CG + row;
                const float rs = rs_mi[mi];
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + mi * kAccStride;
                    float v[32], gt[32];
                    tmem_ld32(lane_addr + c0, v);  // .sync.aligned: every lane, before any divergence
                    if constexpr (DUAL) tmem_ld32(lane_addr + kAccStride + c0, gt);
                    if constexpr (DUAL) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = silu_mul(gt[i], v[i]);
                    }
                    emit(t, c0, v, rs);
                }
            }
        }
    }
    tc_fence_before();
    if constexpr (CG == 2)
        cluster_sync_all();  // the leader's MMAs write the peer's TMEM and commit to its barriers
    else
        __syncthreads();
    if (!DUAL && A.cred) {
        // The S = splits CTAs holding partials of the same rows (cluster ranks
        // x + CG z, z = split) reduce them through DSMEM: split z owns the column
        // slice [z BN/S, (z+1) BN/S), sums the S partials in split order and runs
        // the fused epilogue on it.
        if constexpr (CG == 1) cluster_sync_all();
        if (warp >= 2) {
            const int S = A.splits, cols = BN / S;
            const int z = static_cast<int>(blockIdx.z), row = (warp & 3) * 32 + lane;
            const uint32_t base = smem_u32(smem);
            const float rs = rs_epi;  // (BMT = 1 in the cluster path)
#pragma unroll 1
            for (int c0 = z * cols; c0 < (z + 1) * cols; c0 += 32) {
                float v[32];
#pragma unroll 1
                for (int zz = 0; zz < S; ++zz) {
                    uint32_t a;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                                 : "=r"(a)
                                 : "r"(base + static_cast<uint32_t>(c0 * BM + row) * 4u), "r"(rank + CG * zz));  // same pair half, split zz
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float pv = ld_cluster_f32(a + i * BM * 4);
                        v[i] = zz == 0 ? pv : v[i] + pv;
                    }
                }
                emit(m0 + row, c0, v, rs);
            }
        }
        cluster_sync_all();  // peers have read this CTA's partial
    }
    if (warp == 0) {
        tc_fence_after();
        if constexpr (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kAllocCols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kAllocCols));
    }
}

// ------------------------------------------------------ decode (swap AB) --
// Decode-sized M (<= 64 tokens: the batched engine): the weights are the MMA's
// A operand (M = 128 output rows per CTA, straight from the W tile box) and the
// few token rows its B operand (N = NT), so a stage moves 16 KiB of W and only
// NT x 128 B of X (the 128-row X box of gemm_tc_kernel was 16 KiB of mostly
// zero-filled rows per k-block). D[row][token] lands in TMEM lanes = output
// rows; the epilogue writes y[token][row] coalesced across the lanes.
template <int NT>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float (&v)[NT]) {
    static_assert(NT == 16 || NT == 32, "tcgen05.ld width");
    if constexpr (NT == 32) {
        tmem_ld32(taddr, v);
    } else {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
    }
}

constexpr int kSwapRows = 128;                   // output rows per CTA (the MMA's M)
constexpr int kSwapWBytes = kSwapRows * 128;     // W tile per k-block: 16 KiB

template <int NT, bool DUAL>
__global__ void __launch_bounds__(kThreads, 1) gemm_swap_kernel(const __grid_constant__ TcArgs A) {
    constexpr int kXBytes = NT * 128;
    constexpr int kStage = kSwapWBytes + kXBytes;
    constexpr int kStages = (200 * 1024) / kStage > 12 ? 12 : (200 * 1024) / kStage;
    constexpr uint32_t kGateCol = 64;  // dual: gate accumulator columns [64, 64 + NT)
    constexpr uint32_t kAllocCols = DUAL ? 128 : (NT <= 32 ? 32 : 64);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
    uint64_t* empty = full + kStages;
    uint64_t* tmem_full = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const GemmArgs& g = A.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int tile = blockIdx.y, s = 0;
    if constexpr (!DUAL) {
        while (s + 1 < g.nseg && tile >= A.seg_tiles[s]) {
            tile -= A.seg_tiles[s];
            ++s;
        }
    }
    const GemvSeg& sg = g.seg[s];
    const int n0 = tile * kSwapRows;
    constexpr int kAcc = DUAL ? 2 : 1;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&A.xmap) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kAllocCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    auto seg_of = [&](int j) -> const GemvSeg& { return DUAL ? g.seg[j] : sg; };
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        if (lane == 0) {
            auto kb_range = [&](int j, int& kb0, int& kb1) {
                const int nk = seg_of(j).layout(2).nlines();
                kb0 = nk * static_cast<int>(blockIdx.z) / A.splits;
                kb1 = nk * (static_cast<int>(blockIdx.z) + 1) / A.splits;
            };
            const int t0 = n0 / 16;
            constexpr uint32_t bytes = kStage;
            int npre = 0;  // W tiles of the first ring round, ahead of the grid dependency
            for (int j = 0; j < kAcc && npre < kStages; ++j) {
                int kb0, kb1;
                kb_range(j, kb0, kb1);
                for (int kb = kb0; kb < kb1 && npre < kStages; ++kb, ++npre) {
                    mbar_expect_tx(&full[npre], bytes);
                    tma_load_4d(smem + npre * kStage, &A.wmap[DUAL ? j : s], &full[npre], 0, 0, kb, t0);
                }
            }
            asm volatile("griddepcontrol.wait;" ::: "memory");
            int it = 0;
#pragma unroll 1
            for (int j = 0; j < kAcc; ++j) {
                const GemvSeg& sj = seg_of(j);
                int kb0, kb1;
                kb_range(j, kb0, kb1);
#pragma unroll 1
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    uint8_t* sw = smem + st * kStage;
                    if (it >= npre) {
                        mbar_wait(&empty[st], ph ^ 1);
                        mbar_expect_tx(&full[st], bytes);
                        tma_load_4d(sw, &A.wmap[DUAL ? j : s], &full[st], 0, 0, kb, t0);
                    }
                    tma_load_2d(sw + kSwapWBytes, &A.xmap, &full[st], sj.x_off + kb * BK, 0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16<NT>();  // M = 128 (weights), N = NT (tokens)
            int it = 0;
#pragma unroll 1
            for (int j = 0; j < kAcc; ++j) {
                const int nk = seg_of(j).layout(2).nlines();
                const int kb0 = nk * static_cast<int>(blockIdx.z) / A.splits;
                const int kb1 = nk * (static_cast<int>(blockIdx.z) + 1) / A.splits;
                const uint32_t tacc = tmem_base + static_cast<uint32_t>(j) * kGateCol;
#pragma unroll 1
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int st = it % kStages;
                    const uint32_t ph = (it / kStages) & 1;
                    mbar_wait(&full[st], ph);
                    tc_fence_after();
                    const uint32_t sw = smem_u32(smem + st * kStage);
                    const uint64_t da = sw128_desc(sw), db = sw128_desc(sw + kSwapWBytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc_mma(tacc, da + 2 * k, db + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
                    tc_commit(&empty[st]);
                }
            }
            tc_commit(tmem_full);
        }
    } else {
        // epilogue: warp q holds output rows n0 + 32 q + lane, NT token columns
        const int q = warp & 3;
        const int n = n0 + q * 32 + lane;
        asm volatile("griddepcontrol.wait;" ::: "memory");
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
        float v[NT], gt[NT];
        tmem_ld_cols<NT>(lane_addr, v);
        if constexpr (DUAL) tmem_ld_cols<NT>(lane_addr + kGateCol, gt);
        const bool ok = n < sg.rows;
        const int M = g.M;
        if (!DUAL && A.cred) {
            // cluster split-K: this split's fp32 partial -> own smem as [token][row]
            // (the ring is idle: every MMA that read it has completed)
            float* red = reinterpret_cast<float*>(smem);
#pragma unroll
            for (int t = 0; t < NT; ++t) red[t * kSwapRows + q * 32 + lane] = v[t];
        } else if constexpr (DUAL) {
            if (ok)
#pragma unroll
                for (int t = 0; t < NT; ++t)
                    if (t < M)
                        static_cast<__nv_bfloat16*>(g.y)[static_cast<long long>(t) * g.y_ld + sg.y_off + n] =
                            __float2bfloat16_rn(silu_mul(gt[t], v[t]));
        } else if (A.splits > 1) {
            float* w = g.ws + static_cast<size_t>(blockIdx.z) * M * g.y_ld + sg.y_off + n;
            if (ok)
#pragma unroll
                for (int t = 0; t < NT; ++t)
                    if (t < M) __stcs(w + static_cast<size_t>(t) * g.y_ld, v[t]);
        } else if (g.epi == kGemmStore) {
            if (ok)
#pragma unroll
                for (int t = 0; t < NT; ++t)
                    if (t < M)
                        static_cast<__nv_bfloat16*>(g.y)[static_cast<long long>(t) * g.y_ld + sg.y_off + n] =
                            __float2bfloat16_rn(v[t]);
        } else if (g.epi == kGemmAddF32) {
            if (ok)
#pragma unroll
                for (int t = 0; t < NT; ++t)
                    if (t < M) static_cast<float*>(g.y)[static_cast<long long>(t) * g.y_ld + sg.y_off + n] += v[t];
        } else {  // kGemmQKV: RoPE on row pairs (2i, 2i+1) = adjacent lanes, math.hpp:30-44
            const int ih = n % g.d_head;
            const int p0 = g.p0_dev ? *g.p0_dev : g.p0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const float other = __shfl_xor_sync(0xffffffffu, v[t], 1);
                if (t >= M || !ok) continue;
                const int b = t / g.T, pos = p0 + t % g.T;
                float o = v[t];
                if (sg.epi != kEpiV) {
                    const float2 c = g.rope[static_cast<long long>(pos) * (g.d_head / 2) + (ih >> 1)];
                    o = (ih & 1) ? __fadd_rn(__fmul_rn(other, c.y), __fmul_rn(v[t], c.x))
                                 : __fsub_rn(__fmul_rn(v[t], c.x), __fmul_rn(other, c.y));
                }
                if (sg.epi == kEpiRopeQ) {
                    static_cast<__nv_bfloat16*>(g.y)[static_cast<long long>(t) * g.y_ld + sg.y_off + n] =
                        __float2bfloat16_rn(o);
                } else {
                    const int h = n / g.d_head;
                    __nv_bfloat16* c = static_cast<__nv_bfloat16*>(sg.epi == kEpiRopeK ? g.kcache : g.vcache);
                    c[b * g.cache_bstride + h * g.cache_hstride + static_cast<long long>(pos) * g.d_head + ih] =
                        __float2bfloat16_rn(o);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (!DUAL && A.cred) {
        // The S = splits CTAs of this output tile are one cluster (rank = split).
        // CTA z reduces rows [z R, z R + R) of the tile over all S partials, in
        // split order, straight from the peers' shared memory, and writes them.
        cluster_sync_all();
        if (warp >= 2) {
            const int S = A.splits, R = kSwapRows / S;
            const uint32_t z = cluster_ctarank();
            const int idx = threadIdx.x - 64, r = static_cast<int>(z) * R + idx % R, tg = idx / R;
            const int n = n0 + r;
            const bool ok = n < sg.rows;
            const uint32_t base = smem_u32(smem);
#pragma unroll 1
            for (int t = tg; t < NT; t += S) {
                const uint32_t off = static_cast<uint32_t>(t * kSwapRows + r) * 4u;
                float acc = 0.f;
                for (int zz = 0; zz < S; ++zz) {
                    uint32_t a;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(base + off), "r"(zz));
                    const float pv = ld_cluster_f32(a);
                    acc = zz == 0 ? pv : acc + pv;
                }
                if (!ok || t >= g.M) continue;
                const long long o = static_cast<long long>(t) * g.y_ld + sg.y_off + n;
                if (g.epi == kGemmAddF32)
                    static_cast<float*>(g.y)[o] += acc;
                else
                    static_cast<__nv_bfloat16*>(g.y)[o] = __float2bfloat16_rn(acc);
            }
        }
        cluster_sync_all();  // peers have read this CTA's partial
    }
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kAllocCols));
    }
}

template <int NT, bool DUAL>
void launch_swap(const TcArgs& ta, int tiles, cudaStream_t s) {
    constexpr int kStage = kSwapWBytes + NT * 128;
    constexpr int kStages = (200 * 1024) / kStage > 12 ? 12 : (200 * 1024) / kStage;
    constexpr int kSmem = kStages * kStage + 1024 + 256;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gemm_swap_kernel<NT, DUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        attr = true;
    }
    if (!ta.cred) {
        launch_pdl(gemm_swap_kernel<NT, DUAL>, dim3(1, tiles, ta.splits), dim3(kThreads), kSmem, s, ta);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1, tiles, ta.splits);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = ta.splits;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = std::getenv("FSVD_NO_PDL") ? 1 : 2;
    cudaLaunchKernelEx(&cfg, gemm_swap_kernel<NT, DUAL>, ta);
}

// ------------------------------------------------------------ host side ----
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
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

// Split-K reduction in split order: Y[t][y_off + n] = bf16(sum_z ws[z][t][y_off + n])
// (plain store) or Yf32[t][y_off + n] += sum_z ws[z][...] (residual add).
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const __grid_constant__ TcArgs A) {
    pdl_launch_dependents();
    pdl_wait();
    const GemmArgs& g = A.g;
    const size_t zs = static_cast<size_t>(g.M) * g.y_ld;  // partial stride
    const int t = blockIdx.y;
    const float rs = norm_row_scale(g, t);
    for (int s = 0; s < g.nseg; ++s) {
        const GemvSeg& sg = g.seg[s];
        for (int n = blockIdx.x * 256 + threadIdx.x; n < sg.rows; n += gridDim.x * 256) {
            const size_t c = static_cast<size_t>(t) * g.y_ld + sg.y_off + n;
            // all partials' loads in flight (8 at a time), summed in split order
            float acc = 0.f;
            for (int z0 = 0; z0 < A.splits; z0 += 8) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = z0 + u < A.splits ? __ldcs(g.ws + (z0 + u) * zs + c) : 0.f;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (z0 + u < A.splits) acc = z0 + u == 0 ? v[u] : acc + v[u];
            }
            if (g.epi == kGemmAddF32)
                static_cast<float*>(g.y)[c] += acc;
            else
                static_cast<__nv_bfloat16*>(g.y)[c] = __float2bfloat16_rn(g.norm_ss_in ? acc * rs : acc);
        }
    }
}

template <int BN, bool DUAL, int BMT, int CG = 1>
void launch(const TcArgs& ta, int tiles, int M, cudaStream_t s) {
    using C = Cfg<BN, BMT, CG>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gemm_tc_kernel<BN, DUAL, BMT, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        attr = true;
    }
    dim3 grid((M + BM * BMT * CG - 1) / (BM * BMT * CG) * CG, tiles, ta.splits);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (CG > 1 || ta.cred) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = CG;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = ta.cred ? ta.splits : 1;
        ++na;
    }
    if (!std::getenv("FSVD_NO_PDL")) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, DUAL, BMT, CG>, ta);
    if (ta.splits > 1 && !ta.cred) {
        int rows = 0;
        for (int i = 0; i < ta.g.nseg; ++i) rows = std::max(rows, ta.g.seg[i].rows);
        launch_pdl(splitk_reduce_kernel, dim3((rows + 255) / 256, M), dim3(256), 0, s, ta);
    }
}

}  // namespace

bool gemm_tc_supported(const GemmArgs& a) {
    // X row stride and segment offsets must allow 16 B-aligned TMA boxes
    if (a.x_ld % 8) return false;
    if (a.epi == kGemmQKV && a.d_head % 32) return false;  // the RoPE epilogue's 32-column chunks stay in one head
    for (int i = 0; i < a.nseg; ++i)
        if (a.seg[i].x_off % 8) return false;
    return true;
}

void gemm_tc(const GemmArgs& a, int x_rows, cudaStream_t s) {
    TcArgs ta{};
    ta.g = a;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.x_ld), static_cast<cuuint64_t>(x_rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.x_ld) * 2};
    // decode-sized M: the swap-AB kernel (weights as the MMA's M side)
    // (the QKV epilogue cannot split K: its 96 tiles stream faster as 128 x 256 tiles)
    const bool swap = a.M <= 32 && a.epi != kGemmQKV && !std::getenv("FSVD_NO_SWAP");
    const int NT = a.M <= 16 ? 16 : 32;
    const cuuint32_t box[2] = {BK, static_cast<cuuint32_t>(swap ? NT : BM)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&ta.xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.x), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    const bool dual = a.epi == kGemmSilu;
    auto encode_w = [&](int i, int bn) {
        const WLayout lay = a.seg[i].layout(2);
        const cuuint64_t wd[4] = {64, 16, static_cast<cuuint64_t>(lay.nlines()), static_cast<cuuint64_t>(lay.ntiles())};
        const cuuint64_t ws[3] = {128, static_cast<cuuint64_t>(kLineTileBytes), static_cast<cuuint64_t>(lay.tile_bytes())};
        const cuuint32_t wb[4] = {64, 16, 1, static_cast<cuuint32_t>(bn / 16)};
        const cuuint32_t we[4] = {1, 1, 1, 1};
        const CUresult rw = encode_fn()(&ta.wmap[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a.seg[i].w),
                                        wd, ws, wb, we, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (rw != CUDA_SUCCESS)
            throw std::runtime_error("cuTensorMapEncodeTiled (weights) failed: " + std::to_string(int(rw)));
    };
    const int nseg = dual ? 1 : a.nseg;
    auto count_tiles = [&](int bn) {
        int t = 0;
        for (int i = 0; i < nseg; ++i) t += (a.seg[i].rows + bn - 1) / bn;
        return t;
    };
    int nk_max = 0, nk_min = 1 << 30;
    for (int i = 0; i < a.nseg; ++i) {
        nk_max = std::max(nk_max, a.seg[i].layout(2).nlines());
        nk_min = std::min(nk_min, a.seg[i].layout(2).nlines());
    }
    const bool can_split = !dual && (a.epi == kGemmStore || a.epi == kGemmAddF32) && a.ws;
    if (swap) {
        // 128 output rows per CTA; K split so the CTAs fill one wave (one CTA per
        // SM: ~200 KiB ring), >= 4 k-blocks per split; deterministic in-order reduction
        const int tiles = count_tiles(kSwapRows);
        int sp = 1;
        if (can_split) {
            sp = std::max(1, std::min(148 / tiles, nk_min / 4));
            while (sp > 1 && static_cast<size_t>(sp) * a.M * a.y_ld > a.ws_floats) --sp;
        }
        if (const char* e = std::getenv("FSVD_GEMM_SPLITS"); e && can_split) sp = std::max(1, std::atoi(e));
        // splits reduce in-kernel through DSMEM (one cluster per tile): a power of two <= 8
        ta.cred = sp > 1 && !std::getenv("FSVD_NO_CRED");
        if (ta.cred) sp = sp >= 8 ? 8 : sp >= 4 ? 4 : 2;
        for (int i = 0; i < nseg; ++i) ta.seg_tiles[i] = (a.seg[i].rows + kSwapRows - 1) / kSwapRows;
        for (int i = 0; i < a.nseg; ++i) encode_w(i, kSwapRows);
        ta.splits = sp;
        if (std::getenv("FSVD_GEMM_LOG"))
            std::fprintf(stderr, "gemm_swap M=%d N0=%d nseg=%d nk=%d epi=%d -> NT=%d splits=%d%s tiles=%d\n", a.M,
                         a.seg[0].rows, a.nseg, nk_max, a.epi, NT, sp, ta.cred ? " (cluster)" : "", tiles);
        if (NT == 16) {
            if (dual) launch_swap<16, true>(ta, tiles, s); else launch_swap<16, false>(ta, tiles, s);
        } else {
            if (dual) launch_swap<32, true>(ta, tiles, s); else launch_swap<32, false>(ta, tiles, s);
        }
        if (sp > 1 && !ta.cred) {
            int rows = 0;
            for (int i = 0; i < a.nseg; ++i) rows = std::max(rows, a.seg[i].rows);
            launch_pdl(splitk_reduce_kernel, dim3((rows + 255) / 256, a.M), dim3(256), 0, s, ta);
        }
        return;
    }
    int best_bn = 128, best_sp = 1, best_bmt = 1, best_cg = 1, best_cred = 0;
    if (a.M <= BM) {
        // Decode-sized M (batched engine): the weight stream is the whole cost and
        // the fp32 partials are tiny. Tile width and split-K factor from a wave
        // model: a CTA streams its k-blocks of 16 KiB X + BN x 128 B of W at
        // ~55 GB/s (measured per-SM L2 -> SM rate), CTAs run in waves of 148, a
        // split adds its partials' round trip and a reduction launch.
        constexpr int kBNs[] = {64, 96, 128, 160, 192, 224, 256};
        constexpr double kSmRate = 55e9, kHbm = 6.0e12, kLaunch = 3e-6;
        double best = 1e30;
        for (int bn : kBNs) {
            const int tiles = count_tiles(bn);
            const int max_sp = can_split ? std::max(1, nk_min / 2) : 1;
            for (int sp = 1; sp <= max_sp; ++sp) {
                if (sp > 1 && static_cast<size_t>(sp) * a.M * a.y_ld > a.ws_floats) break;
                const long long ctas = static_cast<long long>(tiles) * sp;
                const double waves = static_cast<double>((ctas + 147) / 148);
                const double kb = (dual ? 2.0 : 1.0) * nk_max / sp;
                double t = waves * kb * (16384.0 + 128.0 * bn) / kSmRate;
                if (sp > 1) t += 2.0 * sp * a.M * a.y_ld * 4.0 / kHbm + kLaunch;
                if (t < best * 0.999) {
                    best = t;
                    best_bn = bn;
                    best_sp = sp;
                }
            }
        }
    } else {
        // Prefill: a wave model fitted to a sweep of every C2 projection shape at
        // M = 512 and 2048 (tools/gemm_sweep.cu, profiles/r1_gemm_sweep.md; median
        // error 9 %, picks within 7.5 % of the best measured config):
        //   t = waves x (2.06 us + 10.22 us/MB x operand bytes per CTA)
        //       + [split] (6.61 us + 0.41 us/MB x fp32 partial bytes)
        // over 128 x {128..256} tiles, 256 x 256 tiles (two TMEM accumulators
        // sharing each W tile) and 1-4 way split K for plain / residual stores.
        constexpr int kBNs[] = {128, 160, 192, 224, 256};
        double best = 1e30;
        for (int bmt = 1; bmt <= (dual ? 1 : 2); ++bmt)
            for (int bn : kBNs) {
                if (bmt == 2 && bn != 256) continue;
                const int tiles = count_tiles(bn);
                const int mt = (a.M + BM * bmt - 1) / (BM * bmt);
                const int max_sp = can_split ? std::max(1, std::min(4, nk_min / 4)) : 1;
                for (int sp = 1; sp <= max_sp; ++sp) {
                    if (sp > 1 && static_cast<size_t>(sp) * a.M * a.y_ld > a.ws_floats) break;
                    const long long ctas = static_cast<long long>(tiles) * mt * sp;
                    const double waves = static_cast<double>((ctas + 147) / 148);
                    const double kb = (dual ? 2.0 : 1.0) * nk_max / sp;
                    const double bytes = kb * (16384.0 * bmt + 128.0 * bn);
                    double t = waves * (2.06 + 10.22 * bytes / 1e6);
                    if (sp > 1) t += 6.61 + 0.41 * sp * static_cast<double>(a.M) * a.y_ld * 8.0 / 1e6;
                    if (t < best * 0.999) {
                        best = t;
                        best_bn = bn;
                        best_sp = sp;
                        best_bmt = bmt;
                    }
                }
            }
    }
    if (a.M > BM && a.M <= 1024 && !dual && !std::getenv("FSVD_NO_PAIR")) {
        // Under-filled long-K projections (qkvA, oA, upgateA, downA at 512 tokens):
        // 256 x 256 CTA-pair tiles, K split over the CTAs of one cluster and
        // reduced through DSMEM (tools/gemm_sweep.cu cred512: 10-20 % faster
        // than the best single-CTA tile at these shapes). S = 4 when that still
        // fits one wave, else 2.
        const int pairs = count_tiles(256) * ((a.M + 255) / 256);
        if (a.epi == kGemmQKV) {  // RoPE / KV-append epilogue: pair tiles, no split (+2 % prefill)
            best_bn = 256;
            best_bmt = 1;
            best_cg = 2;
            best_sp = 1;
        } else if (nk_min >= 32 && pairs * 2 <= 74) {
            best_bn = 256;
            best_bmt = 1;
            best_cg = 2;
            best_sp = pairs * 2 * 4 <= 148 ? 4 : 2;
            best_cred = 1;
        }
    }
    if (const char* e = std::getenv("FSVD_GEMM_BN")) best_bn = std::atoi(e);
    if (const char* e = std::getenv("FSVD_GEMM_SPLITS"); e && can_split) best_sp = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("FSVD_GEMM_BMT"); e && !dual) best_bmt = std::atoi(e) == 2 ? 2 : 1;
    {  // development: per-epilogue override FSVD_GEMM_E<epi>=bn,bmt,splits
        const std::string key = "FSVD_GEMM_E" + std::to_string(a.epi);
        if (const char* e = std::getenv(key.c_str())) {
            int bn = best_bn, bmt = best_bmt, sp = best_sp, cg = best_cg;
            std::sscanf(e, "%d,%d,%d,%d", &bn, &bmt, &sp, &cg);
            best_bn = bn;
            best_bmt = dual ? 1 : (bmt == 2 ? 2 : 1);
            best_sp = can_split ? std::max(1, sp) : 1;
            best_cg = cg == 2 ? 2 : 1;
        }
    }
    if (const char* e = std::getenv("FSVD_GEMM_CG")) best_cg = std::atoi(e) == 2 ? 2 : 1;
    if (a.M <= BM) best_cg = 1;
    // cluster split-K (partials reduced through DSMEM inside the kernel, any epilogue but
    // the dual one): needs one 128-row accumulator, BN/S a multiple of 32, CG*S <= 8
    int cred = best_cred;
    if (const char* e = std::getenv("FSVD_GEMM_CRED")) cred = std::atoi(e);
    if (const char* e = std::getenv(("FSVD_GEMM_E" + std::to_string(a.epi)).c_str())) {
        int x[5] = {0, 0, 0, 0, cred};
        std::sscanf(e, "%d,%d,%d,%d,%d", &x[0], &x[1], &x[2], &x[3], &x[4]);
        cred = x[4];
        if (cred && !dual) best_sp = std::max(1, x[2]);  // cluster splits need no workspace
    }
    if (a.norm_xg) {  // the residual epilogue emits the next RMSNorm's operands: one CTA per output chunk
        best_sp = 1;
        cred = 0;
    }
    if (cred && (dual || best_bmt != 1 || best_sp < 2 || (best_bn % (32 * best_sp)) != 0 || best_cg * best_sp > 8))
        cred = 0;
    if (!cred && !can_split) best_sp = 1;
    ta.cred = cred;
    if (best_bmt == 2) best_bn = 256;
    if (const char* e = std::getenv("FSVD_GEMM_DBG")) ta.dbg = std::atoi(e);
    const int BN = best_bn;
    int tiles = 0;
    for (int i = 0; i < nseg; ++i) {
        ta.seg_tiles[i] = (a.seg[i].rows + BN - 1) / BN;
        tiles += ta.seg_tiles[i];
    }
    ta.splits = best_sp;
    for (int i = 0; i < a.nseg; ++i) encode_w(i, BN / best_cg);  // a pair CTA loads half of the W tile
    if (std::getenv("FSVD_GEMM_LOG"))
        std::fprintf(stderr, "gemm_tc M=%d N0=%d nseg=%d nk=%d epi=%d -> BN=%d BMT=%d CG=%d splits=%d tiles=%d\n",
                     a.M, a.seg[0].rows, a.nseg, nk_max, a.epi, BN, best_bmt, best_cg, best_sp, tiles);
    if (best_bmt == 2) {
        if (best_cg == 2)
            launch<256, false, 2, 2>(ta, tiles, a.M, s);
        else
            launch<256, false, 2>(ta, tiles, a.M, s);
        return;
    }
    if (best_cg == 2) {
#define FSVD_TC_BN2(N)                                   \
    if (BN == N) {                                       \
        if (dual)                                        \
            launch<N, true, 1, 2>(ta, tiles, a.M, s);    \
        else                                             \
            launch<N, false, 1, 2>(ta, tiles, a.M, s);   \
        return;                                          \
    }
        FSVD_TC_BN2(128) FSVD_TC_BN2(160) FSVD_TC_BN2(192) FSVD_TC_BN2(224) FSVD_TC_BN2(256)
#undef FSVD_TC_BN2
    }
#define FSVD_TC_BN(N)                                  \
    if (BN == N) {                                     \
        if (dual)                                      \
            launch<N, true, 1>(ta, tiles, a.M, s);     \
        else                                           \
            launch<N, false, 1>(ta, tiles, a.M, s);    \
        return;                                        \
    }
    FSVD_TC_BN(64) FSVD_TC_BN(96) FSVD_TC_BN(128) FSVD_TC_BN(160) FSVD_TC_BN(192) FSVD_TC_BN(224) FSVD_TC_BN(256)
#undef FSVD_TC_BN
    throw std::runtime_error("gemm_tc: unsupported tile width " + std::to_string(BN));
}

}  // namespace fsvd::k
