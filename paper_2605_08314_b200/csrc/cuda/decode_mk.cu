// Persistent decode megakernel (sm_100a): the whole decode step -- embedding,
// every layer's GEMV chain + attention, head and greedy argmax -- as a list of
// phases executed by one CTA per SM with grid barriers between phases.
//
// Why: a B=1 decode step is ~290 dependent GEMV/attention ops of 1.5-12 us
// each at HBM speed; separate launches leave HBM idle during every ramp and
// tail. Here the weight stream never waits for activations:
//
//  * Weights are in the tile layout (layout.h). A phase's work units are
//    (16-row tile, 8 KiB k-slice) pairs -- one contiguous cp.async.bulk each --
//    split evenly over all warps of the grid (balanced to one unit).
//  * Each warp is its own producer: lane 0 issues the bulk copy (completing
//    on a per-slot mbarrier) of the unit kSlots ahead of the one it computes,
//    walking straight across phase boundaries -- so the next phase's weights
//    are in flight while the warp waits at the grid barrier for activations.
//  * bf16: a unit is reduced on the tensor cores, mma.sync m16n8k16 with the
//    16 weight rows as A and x as B, where x = hi + lo is split into two bf16
//    columns per batch row (fp32-grade activations, bf16 weights, fp32
//    accumulate); a permutation of k inside each 16-wide step makes every
//    A/B fragment load one 8-byte, bank-conflict-free LDS. fp32 weights
//    (parity mode) use an exact CUDA-core dot product.
//  * The grid barrier is the only inter-CTA synchronization. A CTA reduces
//    its units in shared memory and stores one partial sum ("piece") per
//    output tile it touched, in the tile's slot (CTA rank on that tile). The
//    next phase's input staging sums a tile's pieces in slot order and applies
//    the producer's epilogue (RMSNorm scale, residual add, SiLU.mul, RoPE + KV
//    append, logits) -- no in-phase fences, atomics or tickets. Result bits
//    depend only on the grid and the unit split, not on the launch structure,
//    so the eager (one launch per phase), per-layer and full-step plans are
//    bitwise identical.
//  * Attention (decode_mk_attn.cuh) splits the dense cache rows over CTAs.
//
// Reference semantics: SPEC.md:314-322 decode_step; RoPE math.hpp:30-44;
// RMSNorm kernels_scalar.cpp:55-61; SiLU.mul :63-69; argmax (ties -> lowest
// index) math.hpp:132-140.
#include <algorithm>
#include <stdexcept>
#include <utility>
#include <vector>

#include "decode_mk_attn.cuh"
#include "decode_mk_common.cuh"

namespace fsvd::k {
namespace mk {

// ------------------------------------------------------------ unit cursor --
// Units of a phase are numbered 0..total-1: segment by segment, tile-major,
// k-slice fastest; dual phases interleave per tile (up units, then gate
// units). CTA c owns units [total*c/G, total*(c+1)/G); its warps split that
// range. An output tile's pieces are the partial sums of the CTAs whose
// ranges intersect the tile's units (decode_mk.h).
struct SegGeo {
    const char* w;
    int ntiles, nunits, nlines;
    int ubase;  // first unit index of this segment (non-dual)
    int tbase;  // first output tile of this segment
    size_t tile_bytes;
};

template <int ES>
__device__ __forceinline__ SegGeo seg_geo(const GemvSeg& sg, int ubase, int tbase) {
    const WLayout lay = sg.layout(ES);
    SegGeo s;
    s.w = static_cast<const char*>(sg.w);
    s.ntiles = lay.ntiles();
    s.nlines = lay.nlines();
    s.nunits = lay.nunits();
    s.tile_bytes = lay.tile_bytes();
    s.ubase = ubase;
    s.tbase = tbase;
    return s;
}

// Phase geometry (identical for every thread of the CTA).
template <int ES>
struct Geo {
    int nseg, dual, total, cl, ch;  // CTA unit range [cl, ch)
    SegGeo s0, s1, s2;

    __device__ __forceinline__ SegGeo sg(int i) const { return i == 0 ? s0 : (i == 1 ? s1 : s2); }
    __device__ __forceinline__ void init(const MkGemv& g, int cta, int ncta) {
        nseg = g.nseg;
        dual = g.dual;
        s0 = seg_geo<ES>(g.seg[0], 0, 0);
        const int u1 = s0.ntiles * s0.nunits;
        s1 = nseg > 1 ? seg_geo<ES>(g.seg[1], u1, s0.ntiles) : s0;
        const int u2 = nseg > 1 ? u1 + s1.ntiles * s1.nunits : u1;
        s2 = nseg > 2 ? seg_geo<ES>(g.seg[2], u2, s0.ntiles + s1.ntiles) : s0;
        total = dual ? s0.ntiles * (s0.nunits + s1.nunits) : (nseg > 2 ? u2 + s2.ntiles * s2.nunits : u2);
        cl = unit_lo(total, cta, ncta);
        ch = unit_lo(total, cta + 1, ncta);
    }
    // (segment, tile, slice) of unit U
    __device__ __forceinline__ void locate(int U, int& s, int& tile, int& u) const {
        if (dual) {
            const int per = s0.nunits + s1.nunits;
            tile = U / per;
            const int rem = U - tile * per;
            s = rem < s0.nunits ? 0 : 1;
            u = s ? rem - s0.nunits : rem;
        } else {
            s = nseg > 2 && U >= s2.ubase ? 2 : (nseg > 1 && U >= s1.ubase ? 1 : 0);
            const SegGeo c = sg(s);
            const int rel = U - c.ubase;
            tile = rel / c.nunits;
            u = rel - tile * c.nunits;
        }
    }
    // output tile of unit U and that tile's unit range [a, e)
    __device__ __forceinline__ int out_tile(int U, int& a, int& e) const {
        int s, tile, u;
        locate(U, s, tile, u);
        if (dual) {
            const int per = s0.nunits + s1.nunits;
            a = tile * per + (s ? s0.nunits : 0);
            e = s ? (tile + 1) * per : a + s0.nunits;
            return s ? s0.ntiles + tile : tile;
        }
        const SegGeo c = sg(s);
        a = c.ubase + tile * c.nunits;
        e = a + c.nunits;
        return c.tbase + tile;
    }
};

// A warp's position in its own unit stream across the phase program (all
// fields warp-uniform registers; advancing is incremental).
template <int ES>
struct Cursor {
    const MkPhase* phases;
    int p, p_end;
    int U, U_end;    // unit range of this warp in phase p
    int s, tile, u;  // coordinates of unit U
    Geo<ES> geo;
    int cta, ncta, warp;

    __device__ __forceinline__ void enter(int phase) {
        p = phase;
        while (p < p_end && phases[p].kind != kMkGemv) ++p;
        if (p >= p_end) return;
        geo.init(phases[p].g, cta, ncta);
        const int n = geo.ch - geo.cl;
        U = geo.cl + n * warp / kWarpsMk;
        U_end = geo.cl + n * (warp + 1) / kWarpsMk;
        if (U < U_end) geo.locate(U, s, tile, u);
    }
    __device__ __forceinline__ void skip_empty() {
        while (p < p_end && U >= U_end) enter(p + 1);
    }
    __device__ __forceinline__ void init(const MkPhase* ph, int pb, int pe, int c, int nc, int wp) {
        phases = ph;
        p_end = pe;
        cta = c;
        ncta = nc;
        warp = wp;
        U = U_end = 0;
        enter(pb);
        skip_empty();
    }
    __device__ __forceinline__ bool done() const { return p >= p_end; }
    __device__ __forceinline__ int lines() const { return min(kUnitLines, geo.sg(s).nlines - u * kUnitLines); }
    __device__ __forceinline__ int bytes() const { return lines() * kLineTileBytes; }
    __device__ __forceinline__ const char* src() const {
        const SegGeo c = geo.sg(s);
        return c.w + static_cast<size_t>(tile) * c.tile_bytes + static_cast<size_t>(u) * kUnitBytes;
    }
    __device__ __forceinline__ void advance() {
        if (++U >= U_end) {
            enter(p + 1);
            skip_empty();
            return;
        }
        ++u;
        if (geo.dual) {
            if (s == 0 && u == geo.s0.nunits) {
                s = 1;
                u = 0;
            } else if (s == 1 && u == geo.s1.nunits) {
                s = 0;
                u = 0;
                ++tile;
            }
        } else if (u == geo.sg(s).nunits) {
            u = 0;
            if (++tile == geo.sg(s).ntiles) {
                tile = 0;
                ++s;
            }
        }
    }
};

// ---------------------------------------------------------- unit compute --
// 16 row partials of one unit for each batch row -> part[(lu*16 + row)*B + b]
template <typename W, int B>
struct UnitDot;

template <int B>
struct UnitDot<__nv_bfloat16, B> {
    static __device__ __forceinline__ void run(const char* buf, int lines, const Smem& sm, int kbase, int lane,
                                               float* part, int lu) {
        const int g = lane >> 2, t = lane & 3;
        const __nv_bfloat16* xp = static_cast<const __nv_bfloat16*>(sm.x) + g * sm.x_cap;
        float d[4] = {0.f, 0.f, 0.f, 0.f};
        for (int l = 0; l < lines; ++l) {
            const char* lb = buf + l * kLineTileBytes;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int off = ((((2 * j + (t >> 1)) ^ g) & 7) << 4) | ((t & 1) << 3);
                const uint2 r0 = *reinterpret_cast<const uint2*>(lb + g * kLineBytes + off);
                const uint2 r1 = *reinterpret_cast<const uint2*>(lb + (g + 8) * kLineBytes + off);
                uint2 xv = make_uint2(0u, 0u);
                if (g < 2 * B) xv = *reinterpret_cast<const uint2*>(xp + kbase + l * 64 + 16 * j + 4 * t);
                mma_bf16(d, r0.x, r1.x, r0.y, r1.y, xv.x, xv.y);
            }
        }
        if (t < B) {
            part[(lu * 16 + g) * B + t] = d[0] + d[1];
            part[(lu * 16 + g + 8) * B + t] = d[2] + d[3];
        }
    }
};

template <int B>
struct UnitDot<float, B> {
    static __device__ __forceinline__ void run(const char* buf, int lines, const Smem& sm, int kbase, int lane,
                                               float* part, int lu) {
        const int i = lane >> 1, h = lane & 1;
        const float* xf = static_cast<const float*>(sm.x);
        float acc[B];
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] = 0.f;
        for (int l = 0; l < lines; ++l) {
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int c = h * 4 + cc;
                const float4 w = *reinterpret_cast<const float4*>(buf + l * kLineTileBytes + i * kLineBytes +
                                                                  (((c ^ (i & 7)) & 7) << 4));
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const float4 x = *reinterpret_cast<const float4*>(xf + b * sm.x_cap + kbase + l * 32 + c * 4);
                    acc[b] = fmaf(w.x, x.x, acc[b]);
                    acc[b] = fmaf(w.y, x.y, acc[b]);
                    acc[b] = fmaf(w.z, x.z, acc[b]);
                    acc[b] = fmaf(w.w, x.w, acc[b]);
                }
            }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], 1);
            if (h == 0) part[(lu * 16 + i) * B + b] = acc[b];
        }
    }
};

// ---------------------------------------------------------- piece write --
// After the CTA's units are reduced into shared memory: for every output
// tile the CTA touched, sum its units (in unit order) and store the piece in
// the tile's slot = number of non-empty CTAs before this one on the tile.
template <int ES, int B>
__device__ void write_pieces(const MkGemv& g, const Geo<ES>& geo, const float* spart, int tid, int cta, int ncta,
                             const float* inv) {
    const int warp = tid >> 5, lane = tid & 31, i = lane & 15;
    int j = 0;
    for (int U = geo.cl; U < geo.ch; ++j) {
        int a, e;
        const int T = geo.out_tile(U, a, e);
        const int lo = U, hi = min(e, geo.ch);
        U = hi;
        if ((j & (kWarpsMk - 1)) != warp) continue;
        int slot = 0;
        for (int c = unit_cta(a, geo.total, ncta); c < cta; ++c)
            if (unit_lo(geo.total, c + 1, ncta) > unit_lo(geo.total, c, ncta)) ++slot;
        if (lane < 16) {
            float v[B];
#pragma unroll
            for (int b = 0; b < B; ++b) v[b] = 0.f;
            for (int u = lo; u < hi; ++u)
#pragma unroll
                for (int b = 0; b < B; ++b) v[b] += spart[((u - geo.cl) * 16 + i) * B + b];
            float* dst = g.out.base + (static_cast<size_t>(slot) * g.out.R + T * 16 + i) * B;
#pragma unroll
            for (int b = 0; b < B; ++b) dst[b] = v[b] * inv[b];
        }
    }
}

// ------------------------------------------------------------ GEMV phase --
template <typename W, int B>
__device__ __forceinline__ void gemv_phase(const MkPhase& ph, int phase_idx, Smem sm, int tid, int cta,
                                           int ncta, Cursor<sizeof(W)>& cs, Cursor<sizeof(W)>& is,
                                           Cursor<sizeof(W)>& pf, uint32_t& seq, uint64_t policy,
                                           unsigned long long* tr) {
    constexpr int ES = sizeof(W);
    const MkGemv& g = ph.g;
    // this phase's carve of the shared region: x planes (stride x_len), then unit partials
    sm.x_cap = g.x_len;
    sm.part = reinterpret_cast<float*>(static_cast<char*>(sm.x) +
                                       ((static_cast<size_t>(B) * XPlanes<W>::kPlanes * g.x_len * ES + 15) & ~size_t(15)));
    stage_x<W, B>(g, sm, tid, cta, ncta);
    if (tr && tid == 0) tr[2] = gtimer();
    float inv[B];
#pragma unroll
    for (int b = 0; b < B; ++b) inv[b] = sm.misc[128 + b];
    const int warp = tid >> 5, lane = tid & 31;
    Geo<ES> geo;
    geo.init(g, cta, ncta);
    while (!cs.done() && cs.p == phase_idx) {
        const uint32_t slot = seq % kSlots, par = (seq / kSlots) & 1u;
        uint64_t* bar = sm.full + warp * kSlots + slot;
        char* buf = sm.slots + (static_cast<size_t>(warp) * kSlots + slot) * kUnitBytes;
        mbar_wait(bar, par);
        const int kbase = g.seg[cs.s].x_off + cs.u * kUnitLines * (kLineBytes / ES);
        UnitDot<W, B>::run(buf, cs.lines(), sm, kbase, lane, sm.part, cs.U - geo.cl);
        __syncwarp();
        // refill this slot with the unit kSlots ahead (possibly in a later phase)
        if (!is.done()) {
            if (lane == 0) {
                fence_proxy_async();
                mbar_expect_tx(bar, static_cast<uint32_t>(is.bytes()));
                bulk_g2s(buf, is.src(), static_cast<uint32_t>(is.bytes()), bar, policy);
            }
            is.advance();
        }
        // keep HBM busy through the phase overheads: L2 prefetch further ahead
        if (!pf.done()) {
            if (lane == 0) prefetch_l2_bulk(pf.src(), static_cast<uint32_t>(pf.bytes()));
            pf.advance();
        }
        ++seq;
        cs.advance();
    }
    if (tr && lane == 0) tr[4 + (warp & 1)] = gtimer();  // units done: warps 0 and 1
    __syncthreads();
    if (tr && tid == 0) tr[6] = gtimer();
    write_pieces<ES, B>(g, geo, sm.part, tid, cta, ncta, inv);
    if (tr && tid == 0) tr[7] = gtimer();
}

// ---------------------------------------------------------- argmax phase --
// logits = sum of the head pieces; per-CTA best (ties -> lowest index,
// math.hpp:132-140); the last CTA (ticket) reduces the CTA bests in CTA order,
// sets the next input token and advances the length register.
template <int B>
__device__ void argmax_phase(const MkArgmax& m, const Smem& sm, int tid, int cta, int ncta) {
    const int warp = tid >> 5, lane = tid & 31;
    const int r0 = unit_lo(m.vocab, cta, ncta), r1 = unit_lo(m.vocab, cta + 1, ncta);
    float* sv = sm.misc;                                       // [warps][B]
    int* si = reinterpret_cast<int*>(sm.misc + kWarpsMk * 4);  // [warps][B]
    for (int b = 0; b < B; ++b) {
        float bv = -CUDART_INF_F;
        int bi = 0x7fffffff;
        for (int r = r0 + tid; r < r1; r += kThreadsMk) {
            const float v = piece_sum<B>(m.pc, r, b);
            m.logits[static_cast<long long>(b) * m.vocab + r] = v;
            if (better(v, r, bv, bi)) {
                bv = v;
                bi = r;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (better(ov, oi, bv, bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            sv[warp * 4 + b] = bv;
            si[warp * 4 + b] = bi;
        }
    }
    __syncthreads();
    __shared__ unsigned last;
    if (tid == 0) {
        for (int b = 0; b < B; ++b) {
            float bv = -CUDART_INF_F;
            int bi = 0x7fffffff;
            for (int w = 0; w < kWarpsMk; ++w)
                if (better(sv[w * 4 + b], si[w * 4 + b], bv, bi)) {
                    bv = sv[w * 4 + b];
                    bi = si[w * 4 + b];
                }
            m.best_v[cta * B + b] = bv;
            m.best_i[cta * B + b] = bi;
        }
        __threadfence();
        last = atomicAdd(m.ticket, 1u) + 1u == static_cast<unsigned>(ncta);
        if (last) __threadfence();
    }
    __syncthreads();
    if (!last || warp != 0) return;
    for (int b = 0; b < B; ++b) {
        float bv = -CUDART_INF_F;
        int bi = 0x7fffffff;
        for (int c = lane; c < ncta; c += 32) {
            const float v = __ldcg(m.best_v + c * B + b);
            const int i = __ldcg(m.best_i + c * B + b);
            if (better(v, i, bv, bi)) {
                bv = v;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (better(ov, oi, bv, bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            if (bi == 0x7fffffff) bi = 0;
            m.tokens[b] = bi;
            if (m.out) m.out[static_cast<long long>(b) * m.out_ld + *m.step] = bi;
        }
    }
    if (lane == 0) {
        *m.pos += m.pos_inc;
        *m.step += 1;
        *m.ticket = 0u;
    }
}

// ----------------------------------------------------------- the kernel --
template <typename W, int B, int DH>
__global__ void __launch_bounds__(kThreadsMk, 1) decode_mk_kernel(const MkPhase* __restrict__ phases, int p_begin,
                                                                  int p_end, unsigned* bar, int region_bytes,
                                                                  int red_floats, unsigned long long* trace) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    constexpr int ES = sizeof(W);
    Smem sm;
    sm.slots = reinterpret_cast<char*>(smem_raw);
    sm.full = reinterpret_cast<uint64_t*>(smem_raw + static_cast<size_t>(kWarpsMk) * kSlots * kUnitBytes);
    sm.x = sm.full + kWarpsMk * kSlots;
    sm.x_cap = 0;
    sm.part = nullptr;  // carved per phase (gemv_phase)
    sm.red = reinterpret_cast<float*>(static_cast<char*>(sm.x) + region_bytes);
    sm.misc = sm.red + red_floats;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, cta = blockIdx.x, ncta = gridDim.x;
    if (tid < kWarpsMk * kSlots) mbar_init(&sm.full[tid], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    // per-warp unit streams: compute (cs), bulk-copy issue (is, kSlots ahead), L2 prefetch (pf)
    Cursor<ES> cs, is, pf;
    cs.init(phases, p_begin, p_end, cta, ncta, warp);
    is.init(phases, p_begin, p_end, cta, ncta, warp);
    pf.init(phases, p_begin, p_end, cta, ncta, warp);
    const uint64_t policy = evict_first_policy();
    uint32_t seq = 0;
    for (int sl = 0; sl < kSlots && !is.done(); ++sl) {
        if (lane == 0) {
            uint64_t* b = sm.full + warp * kSlots + sl;
            mbar_expect_tx(b, static_cast<uint32_t>(is.bytes()));
            bulk_g2s(sm.slots + (static_cast<size_t>(warp) * kSlots + sl) * kUnitBytes, is.src(),
                     static_cast<uint32_t>(is.bytes()), b, policy);
        }
        is.advance();
    }
    for (int k = 0; k < kSlots + kPrefetch && !pf.done(); ++k) {
        if (k >= kSlots && lane == 0) prefetch_l2_bulk(pf.src(), static_cast<uint32_t>(pf.bytes()));
        pf.advance();
    }

    const int nph = p_end - p_begin;
    for (int p = p_begin; p < p_end; ++p) {
        const int idx = p - p_begin;
        unsigned long long* tr = trace ? trace + (static_cast<size_t>(cta) * nph + idx) * 8 : nullptr;
        if (tr && tid == 0) tr[0] = gtimer();
        const MkPhase& ph = phases[p];
        // the history of the coming attention is immutable: prefetch it to L2
        if (ph.kind == kMkGemv && p + 2 < p_end && phases[p + 2].kind == kMkAttn && phases[p + 1].kind == kMkGemv)
            attn_prefetch<W, B, DH>(phases[p + 2].a, tid, cta, ncta);
        if (idx > 0) {  // grid barrier: all CTAs finished phase idx-1
            if (tid == 0) {
                const unsigned target = static_cast<unsigned>(idx) * ncta;
                while (ld_acquire(bar) < target) __nanosleep(20);
            }
            __syncthreads();
        }
        if (tr && tid == 0) tr[1] = tr[2] = tr[4] = tr[5] = tr[6] = tr[7] = gtimer();
        switch (ph.kind) {
            case kMkGemv:
                gemv_phase<W, B>(ph, p, sm, tid, cta, ncta, cs, is, pf, seq, policy, tr);
                break;
            case kMkAttn:
                attn_phase<W, B, DH>(ph.a, sm, tid, cta, ncta);
                break;
            case kMkArgmax:
                argmax_phase<B>(ph.m, sm, tid, cta, ncta);
                break;
            default:
                break;
        }
        // arrive: this CTA's writes of phase idx are complete
        __syncthreads();
        if (tr && tid == 0) tr[3] = gtimer();
        if (tid == 0) {
            __threadfence();
            const unsigned v = atomicAdd(bar, 1u) + 1u;
            if (v == static_cast<unsigned>(nph) * ncta) *bar = 0u;  // last arrival of the launch: reset
        }
    }
}

template <typename W, int B, int DH>
void launch_t(const MkLaunch& L, cudaStream_t s) {
    auto fn = decode_mk_kernel<W, B, DH>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem_bytes);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(L.grid);
    cfg.blockDim = dim3(kThreadsMk);
    cfg.dynamicSmemBytes = L.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, fn, L.phases, L.p_begin, L.p_end, L.bar, L.region_bytes, L.red_floats, L.trace);
}

}  // namespace mk

// --------------------------------------------------------- host mirrors --
namespace {
struct HostSeg {
    int ntiles, nunits;
};
HostSeg host_seg(const GemvSeg& s, int es) {
    const WLayout l = s.layout(es);
    return {l.ntiles(), l.nunits()};
}
long long ulo(long long total, int c, int G) { return total * c / G; }
}  // namespace

int mk_units(const GemvSeg* seg, int nseg, int dual, int esize) {
    if (dual) {
        const HostSeg a = host_seg(seg[0], esize), b = host_seg(seg[1], esize);
        return a.ntiles * (a.nunits + b.nunits);
    }
    int t = 0;
    for (int s = 0; s < nseg; ++s) {
        const HostSeg h = host_seg(seg[s], esize);
        t += h.ntiles * h.nunits;
    }
    return t;
}

int mk_out_tiles(const GemvSeg* seg, int nseg, int dual, int esize) {
    if (dual) return 2 * host_seg(seg[0], esize).ntiles;
    int t = 0;
    for (int s = 0; s < nseg; ++s) t += host_seg(seg[s], esize).ntiles;
    return t;
}

int mk_npieces(const GemvSeg* seg, int nseg, int dual, int esize, int grid, uint8_t* npieces) {
    const long long total = mk_units(seg, nseg, dual, esize);
    // unit ranges of the output tiles, in output-tile order
    std::vector<std::pair<long long, long long>> rng;
    if (dual) {
        const HostSeg a = host_seg(seg[0], esize), b = host_seg(seg[1], esize);
        const long long per = a.nunits + b.nunits;
        for (int t = 0; t < a.ntiles; ++t) rng.push_back({t * per, t * per + a.nunits});
        for (int t = 0; t < a.ntiles; ++t) rng.push_back({t * per + a.nunits, (t + 1) * per});
    } else {
        long long ub = 0;
        for (int s = 0; s < nseg; ++s) {
            const HostSeg h = host_seg(seg[s], esize);
            for (int t = 0; t < h.ntiles; ++t) rng.push_back({ub + t * h.nunits, ub + (t + 1) * h.nunits});
            ub += static_cast<long long>(h.ntiles) * h.nunits;
        }
    }
    int mx = 0;
    for (size_t T = 0; T < rng.size(); ++T) {
        int n = 0;
        for (int c = 0; c < grid; ++c) {
            const long long lo = std::max(ulo(total, c, grid), rng[T].first);
            const long long hi = std::min(ulo(total, c + 1, grid), rng[T].second);
            if (lo < hi) ++n;
        }
        if (n > 255) throw std::runtime_error("decode megakernel: more than 255 pieces on one tile");
        npieces[T] = static_cast<uint8_t>(n);
        mx = std::max(mx, n);
    }
    return mx;
}

int mk_region_bytes(int batch, WType wt, int x_len, int units_per_cta) {
    const int es = wt == kBF16 ? 2 : 4, planes = wt == kBF16 ? 2 : 1;
    return ((batch * planes * x_len * es + 15) & ~15) + units_per_cta * 16 * batch * 4;
}

int mk_red_floats(int batch, int n_heads, int d_head) {
    return (std::max(mk::kWarpsMk * (d_head + 2), 3 * batch * n_heads) + 31) / 32 * 32;
}

int mk_smem_bytes(int region_bytes, int red_floats) {
    return mk::kWarpsMk * mk::kSlots * kUnitBytes + mk::kWarpsMk * mk::kSlots * 8 + region_bytes + red_floats * 4 +
           256 * 4 + 128;
}

int mk_warps() { return mk::kWarpsMk; }

bool mk_launch(WType wt, int batch, int d_head, const MkLaunch& L, cudaStream_t s) {
#define FSVD_MK(W, BB, DHH) \
    if (batch == BB && d_head == DHH) { mk::launch_t<W, BB, DHH>(L, s); return true; }
    if (wt == kBF16) {
        FSVD_MK(__nv_bfloat16, 1, 128) FSVD_MK(__nv_bfloat16, 2, 128) FSVD_MK(__nv_bfloat16, 1, 64)
        FSVD_MK(__nv_bfloat16, 2, 64) FSVD_MK(__nv_bfloat16, 1, 32) FSVD_MK(__nv_bfloat16, 2, 32)
    } else {
        FSVD_MK(float, 1, 128) FSVD_MK(float, 2, 128) FSVD_MK(float, 1, 64) FSVD_MK(float, 2, 64)
        FSVD_MK(float, 1, 32) FSVD_MK(float, 2, 32)
    }
#undef FSVD_MK
    return false;
}

}  // namespace fsvd::k
