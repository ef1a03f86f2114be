// Shared pieces of the decode megakernel: PTX wrappers, the work split
// (host + device), and the tensor-core chunk reduction.
#pragma once

#include <math_constants.h>

#include "common.cuh"
#include "decode_mk.h"
#include "kernels.h"

namespace fsvd::k::mk {

using namespace fsvd::dev;

constexpr int kConsumerWarps = 8;
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kThreads = kConsumerThreads + 32;  // + the producer warp

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerThreads) : "memory");
}
// D(16x8, f32) += A(16x16, bf16, row) * B(16x8, bf16, col)
__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) { return v > bv || (v == bv && i < bi); }

}  // namespace fsvd::k::mk

namespace fsvd::k {

// ------------------------------------------------------------ work split --
// Units of a GEMV phase are (16-row tile, 128-byte line) pairs numbered
// segment by segment, tile-major, line-fastest; a dual phase interleaves per
// tile: the up tile's lines, then the gate tile's. A "run" is the unit span
// of one (output tile, sub) -- sub 1 = the gate half of a dual tile. CTA c
// of G owns units [total*c/G, total*(c+1)/G); its chunks are <= kChunkLines
// units of one run, starting at the run start or at the CTA's first unit.
// All arithmetic is 32-bit (total * G < 2^32); the per-chunk walk is
// incremental (ChunkIter) -- no divisions on the streaming path.
struct MkSplit {
    int total;
    int nseg, dual;
    int ubase[3];
    int ntiles[3], nlines[3], tbase[3];
    int out_tiles;
    int exact;  // 1: even unit split (tiles may be shared by CTAs: pieces exchange)

    FSVD_HD void init(const GemvSeg* seg, int nseg_, int dual_, int es, int exact_ = 0) {
        nseg = nseg_;
        dual = dual_;
        exact = exact_;
        int u = 0, t = 0;
        for (int s = 0; s < 3; ++s) {
            ntiles[s] = nlines[s] = tbase[s] = 0;
            ubase[s] = u;
            if (s >= nseg) continue;
            const WLayout l = seg[s].layout(es);
            ntiles[s] = l.ntiles();
            nlines[s] = l.nlines();
            tbase[s] = t;
            if (!dual) {
                u += ntiles[s] * nlines[s];
                t += ntiles[s];
            }
        }
        if (dual) {
            total = ntiles[0] * (nlines[0] + nlines[1]);
            out_tiles = ntiles[0];
        } else {
            total = u;
            out_tiles = t;
        }
    }
    FSVD_HD int subs() const { return dual ? 2 : 1; }
    // First unit of CTA c: the even split total*c/G snapped to the nearest
    // output-tile boundary, so every tile has exactly one owner (no cross-CTA
    // reduction). The imbalance this leaves is absorbed by HBM sharing: a CTA
    // with one tile more pulls more bandwidth while the others idle.
    FSVD_HD int lo(int c, int G) const {
        if (c <= 0) return 0;
        if (c >= G) return total;
        const int U = static_cast<int>(static_cast<unsigned>(total) * static_cast<unsigned>(c) / static_cast<unsigned>(G));
        if (exact) return U;
        int a, e;
        tile_span(tile_of(U), a, e);
        return U - a <= e - U ? a : e;
    }
    FSVD_HD int seg_of_tile(int T) const {
        int s = 0;
        if (!dual)
            while (s + 1 < nseg && T >= tbase[s + 1]) ++s;
        return s;
    }
    // unit span of output tile T (both subs for dual)
    FSVD_HD void tile_span(int T, int& a, int& e) const {
        if (dual) {
            const int per = nlines[0] + nlines[1];
            a = T * per;
            e = a + per;
            return;
        }
        const int s = seg_of_tile(T);
        a = ubase[s] + (T - tbase[s]) * nlines[s];
        e = a + nlines[s];
    }
    // unit span of run (T, sub)
    FSVD_HD void run_span(int T, int sub, int& a, int& e) const {
        tile_span(T, a, e);
        if (dual) {
            if (sub == 0)
                e = a + nlines[0];
            else
                a += nlines[0];
        }
    }
    // output tile of unit U
    FSVD_HD int tile_of(int U) const {
        if (dual) return U / (nlines[0] + nlines[1]);
        int s = 0;
        while (s + 1 < nseg && U >= ubase[s + 1]) ++s;
        return tbase[s] + (U - ubase[s]) / nlines[s];
    }
    // CTA owning unit U (non-empty range)
    FSVD_HD int cta_of(int U, int G) const {
        int c = static_cast<int>(static_cast<unsigned>(U) * static_cast<unsigned>(G) / static_cast<unsigned>(total));
        if (c >= G) c = G - 1;
        while (c + 1 < G && lo(c + 1, G) <= U) ++c;
        while (c > 0 && lo(c, G) > U) --c;
        return c;
    }
    // number of non-empty CTAs in [c0, c1)
    FSVD_HD int nonempty(int c0, int c1, int G) const {
        int n = 0;
        int l = lo(c0, G);
        for (int c = c0; c < c1; ++c) {
            const int h = lo(c + 1, G);
            n += h > l;
            l = h;
        }
        return n;
    }
    // chunks of run span [a, e) inside [ulo, uhi)
    static FSVD_HD int run_chunks(int a, int e, int ulo, int uhi) {
        const int x = a > ulo ? a : ulo, y = e < uhi ? e : uhi;
        return y > x ? (y - x + kChunkLines - 1) / kChunkLines : 0;
    }
};

// Incremental walk over one CTA's chunks of a phase (shared by the producer
// and the consumers, so both see the same chunk sequence).
struct ChunkIter {
    int U, uhi;
    int s, t, line;  // segment (dual: sub), tile within segment, line within run
    FSVD_HD void begin(const MkSplit& sp, int ulo, int uhi_) {
        U = ulo;
        uhi = uhi_;
        if (U >= uhi) return;
        if (sp.dual) {
            const int per = sp.nlines[0] + sp.nlines[1];
            t = U / per;
            const int rem = U - t * per;
            s = rem < sp.nlines[0] ? 0 : 1;
            line = s ? rem - sp.nlines[0] : rem;
        } else {
            s = 0;
            while (s + 1 < sp.nseg && U >= sp.ubase[s + 1]) ++s;
            const int rel = U - sp.ubase[s];
            t = rel / sp.nlines[s];
            line = rel - t * sp.nlines[s];
        }
    }
    FSVD_HD bool done() const { return U >= uhi; }
    // lines of the current chunk
    FSVD_HD int lines(const MkSplit& sp) const {
        int n = sp.nlines[s] - line;
        if (n > kChunkLines) n = kChunkLines;
        if (n > uhi - U) n = uhi - U;
        return n;
    }
    FSVD_HD void advance(const MkSplit& sp, int nl) {
        U += nl;
        line += nl;
        if (line < sp.nlines[s]) return;
        line = 0;
        if (sp.dual) {
            if (s == 0) {
                s = 1;
            } else {
                s = 0;
                ++t;
            }
        } else if (++t == sp.ntiles[s]) {
            t = 0;
            ++s;
        }
    }
};

// A CTA's chunk sequence in "boundary tiles first" order: the first tile of
// its range, then the last, then the interior -- so the per-CTA partials of
// the two tiles shared with neighbouring CTAs are exchanged while the
// interior still streams. Every tile's chunks stay contiguous.
struct ChunkSeq {
    int r_lo[3], r_hi[3];
    int nr, r;
    ChunkIter it;
    int c_run;  // chunk index inside the current run
    FSVD_HD void begin(const MkSplit& sp, int ulo, int uhi) {
        nr = 0;
        if (ulo < uhi) {
            const int Tf = sp.tile_of(ulo), Tl = sp.tile_of(uhi - 1);
            int a, e, a2, e2;
            sp.tile_span(Tf, a, e);
            sp.tile_span(Tl, a2, e2);
            const int ef = e < uhi ? e : uhi;
            r_lo[nr] = ulo; r_hi[nr] = ef; ++nr;
            if (Tl > Tf) {
                r_lo[nr] = a2; r_hi[nr] = uhi; ++nr;
                if (a2 > ef) { r_lo[nr] = ef; r_hi[nr] = a2; ++nr; }
            }
        }
        r = 0;
        c_run = 0;
        if (nr) it.begin(sp, r_lo[0], r_hi[0]);
        else it.U = it.uhi = 0;
    }
    FSVD_HD bool done() const { return r >= nr; }
    FSVD_HD int tile(const MkSplit& sp) const { return sp.dual ? it.t : sp.tbase[it.s] + it.t; }
    FSVD_HD int sub(const MkSplit& sp) const { return sp.dual ? it.s : 0; }
    // advance past the current chunk of nl lines
    FSVD_HD void advance(const MkSplit& sp, int nl) {
        const int line0 = it.line;
        it.advance(sp, nl);
        (void)line0;
        c_run = it.line == 0 ? 0 : c_run + 1;
        if (it.done()) {
            ++r;
            c_run = 0;
            if (r < nr) it.begin(sp, r_lo[r], r_hi[r]);
        }
    }
};

// Same split over a plain row space (attention: B*H*len key rows). 32-bit
// products on purpose (64-bit divides are emulated and measured 16% slower on
// the decode step); Session rejects shapes with B*H*capacity*grid >= 2^32.
struct RowSplit {
    int total;
    FSVD_HD int lo(int c, int G) const {
        return static_cast<int>(static_cast<unsigned>(total) * static_cast<unsigned>(c) / static_cast<unsigned>(G));
    }
    FSVD_HD int cta_of(int U, int G) const {
        int c = static_cast<int>(static_cast<unsigned>(U) * static_cast<unsigned>(G) / static_cast<unsigned>(total));
        if (c >= G) c = G - 1;
        while (c + 1 < G && lo(c + 1, G) <= U) ++c;
        while (c > 0 && lo(c, G) > U) --c;
        return c;
    }
    FSVD_HD int nonempty(int c0, int c1, int G) const {
        int n = 0;
        int l = lo(c0, G);
        for (int c = c0; c < c1; ++c) {
            const int h = lo(c + 1, G);
            n += h > l;
            l = h;
        }
        return n;
    }
};

}  // namespace fsvd::k

namespace fsvd::k::mk {

// ---------------------------------------------------------- chunk compute --
// 16 row partials of one chunk (nl lines of a tile) for each batch row ->
// rec[(row)*B + b]. bf16: tensor cores, mma.sync m16n8k16 with the 16
// weight rows as A and the staged x planes as B (column 2b = hi, 2b+1 = lo);
// k is permuted inside each 16-wide step so that every A and B fragment is
// one 8-byte, bank-conflict-free shared load (the XOR swizzle of layout.h).
template <typename W, int B>
struct ChunkDot;

template <int B>
struct ChunkDot<__nv_bfloat16, B> {
    // A fragments by ldmatrix.x4 straight from the swizzled line tile (each
    // 8x8 matrix = 8 rows x 16 B at distinct XOR-swizzled chunks: conflict-free),
    // B fragments = 4-byte pairs of the staged x planes.
    static __device__ __forceinline__ void run(const char* buf, int nl, const __nv_bfloat16* x, int x_len, int kbase,
                                               int lane, float* rec) {
        const int g = lane >> 2, t = lane & 3;
        const int r = (lane & 7) + 8 * ((lane >> 3) & 1);  // row this lane addresses for ldmatrix
        const int hi = lane >> 4;                          // which 16-B chunk of the k-step
        // the planes are k-permuted per 64-element line (plane_pos): lane t's B
        // fragments of the line's four k-steps are 32 contiguous bytes
        const __nv_bfloat16* xp = x + g * x_len + kbase + 16 * t;
        const uint32_t a_row = static_cast<uint32_t>(__cvta_generic_to_shared(buf)) + r * kLineBytes;
        // two accumulator sets (even / odd lines): the per-accumulator mma chain is
        // half as long
        float d[2][4][4] = {};
        auto line = [&](int l, float (&dd)[4][4]) {
            const uint32_t lrow = a_row + l * kLineTileBytes;
            uint4 xb[2] = {make_uint4(0u, 0u, 0u, 0u), make_uint4(0u, 0u, 0u, 0u)};
            if (g < 2 * B) {
                xb[0] = *reinterpret_cast<const uint4*>(xp + l * 64);
                xb[1] = *reinterpret_cast<const uint4*>(xp + l * 64 + 8);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t a0, a1, a2, a3;
                const uint32_t addr = lrow + ((((2 * j + hi) ^ r) & 7) << 4);
                asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                             : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                             : "r"(addr));
                const uint4& q = xb[j >> 1];
                const uint32_t b0 = (j & 1) ? q.z : q.x, b1 = (j & 1) ? q.w : q.y;
                mma_bf16(dd[j], a0, a1, a2, a3, b0, b1);
            }
        };
        int l = 0;
#pragma unroll 1
        for (; l + 1 < nl; l += 2) {
            line(l, d[0]);
            line(l + 1, d[1]);
        }
        if (l < nl) line(l, d[0]);
        if (t < B) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                s0 += ((d[p][0][0] + d[p][1][0]) + (d[p][2][0] + d[p][3][0])) +
                      ((d[p][0][1] + d[p][1][1]) + (d[p][2][1] + d[p][3][1]));
                s1 += ((d[p][0][2] + d[p][1][2]) + (d[p][2][2] + d[p][3][2])) +
                      ((d[p][0][3] + d[p][1][3]) + (d[p][2][3] + d[p][3][3]));
            }
            rec[g * B + t] = s0;
            rec[(g + 8) * B + t] = s1;
        }
    }
};

// fp32 weights (parity mode): exact CUDA-core dot, 2 lanes per row
template <int B>
struct ChunkDot<float, B> {
    static __device__ __forceinline__ void run(const char* buf, int nl, const float* x, int x_len, int kbase, int lane,
                                               float* rec) {
        const int i = lane >> 1, h = lane & 1;
        float acc[B];
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] = 0.f;
        for (int l = 0; l < nl; ++l) {
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int c = h * 4 + cc;
                const float4 w = *reinterpret_cast<const float4*>(buf + l * kLineTileBytes + i * kLineBytes +
                                                                  (((c ^ (i & 7)) & 7) << 4));
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const float4 xv = *reinterpret_cast<const float4*>(x + b * x_len + kbase + l * 32 + c * 4);
                    acc[b] = fmaf(w.x, xv.x, acc[b]);
                    acc[b] = fmaf(w.y, xv.y, acc[b]);
                    acc[b] = fmaf(w.z, xv.z, acc[b]);
                    acc[b] = fmaf(w.w, xv.w, acc[b]);
                }
            }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], 1);
            if (h == 0) rec[i * B + b] = acc[b];
        }
    }
};

// ------------------------------------------------------- planes writers --
template <typename W>
struct PlaneIO;
template <>
struct PlaneIO<__nv_bfloat16> {
    static constexpr int kBytesPerElem = 4;  // hi + lo
    // Element k of each 64-element line sits at 16 t + 4 j + w, where j = k / 16
    // is the mma k-step, t = (k % 8) / 2 the lane quad index and w picks
    // (2t, 2t+1, 2t+8, 2t+9): the B fragments lane t needs for the whole line.
    static __device__ __forceinline__ int plane_pos(int i) {
        const int k = i & 63, j = k >> 4, r = k & 15;
        return (i & ~63) | (((r & 7) >> 1) << 4) | (j << 2) | (r & 1) | ((r & 8) >> 2);
    }
    static __device__ __forceinline__ void put(const Planes& p, int b, int i, float v) {
        __nv_bfloat16* q = static_cast<__nv_bfloat16*>(p.p) + static_cast<size_t>(2 * b) * p.len;
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        const int o = plane_pos(i);
        q[o] = h;
        q[p.len + o] = __float2bfloat16_rn(v - __bfloat162float(h));
    }
};
template <>
struct PlaneIO<float> {
    static constexpr int kBytesPerElem = 4;
    static __device__ __forceinline__ void put(const Planes& p, int b, int i, float v) {
        static_cast<float*>(p.p)[static_cast<size_t>(b) * p.len + i] = v;
    }
};

}  // namespace fsvd::k::mk
