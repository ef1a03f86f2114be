// Persistent decode megakernel (sm_100a): the whole decode step -- embedding,
// every layer's low-rank GEMV chain and attention, head and greedy argmax --
// as a list of phases executed by one CTA per SM, grid barriers between
// phases (SPEC.md:314-322 decode_step).
//
// Why: a B=1 decode step is ~290 dependent GEMV / attention ops of 1.5-12 us
// each at HBM speed; separate kernels leave HBM idle during every launch ramp
// and tail. Here the weight stream never waits for activations:
//
//  * Producer warp (one per CTA): walks the GEMV phases of the launch in
//    order and streams this CTA's weight units through a shared-memory ring
//    of 22 KiB chunks with cp.async.bulk (mbarrier complete_tx), gated only
//    by free ring slots -- across phase boundaries, so the next phase's
//    weights land while the consumers wait at the grid barrier.
//  * Consumer warps (8): per GEMV phase, one bulk copy stages the input
//    vector (ready-made hi/lo bf16 planes, written by the previous phase's
//    finalizers); chunk j of the phase goes to warp j % 8, which reduces it on
//    the tensor cores (mma.sync, fp32 accumulate) into a per-chunk record.
//  * Finalize: the CTA sums the records of each output tile in chunk order;
//    a tile shared with neighbouring CTAs goes through per-CTA pieces and a
//    per-tile counter, and its last contributor sums the pieces in CTA order
//    and applies the epilogue (RMSNorm scale, RoPE + KV append, residual add,
//    SiLU.mul, logits) -- once per row, deterministic for any launch split.
//  * Attention (dense KV): the B*H*len key rows are split
//    evenly over the CTAs, online softmax per warp (math.hpp:56-101), merged
//    per head by its last contributor into the o-projection's input planes.
//
// Reference semantics: RoPE math.hpp:30-44 (interleaved pairs, host-double
// angles); RMSNorm kernels_scalar.cpp:55-61; SiLU.mul :63-69; argmax ties ->
// lowest index math.hpp:132-140.
#include <algorithm>
#include <stdexcept>
#include <vector>

#include "decode_mk_common.cuh"

namespace fsvd::k {
namespace mk {

// full[stages], empty[stages], xbar, abar -- rounded up to 128 B
__host__ __device__ constexpr int mk_barrier_bytes(int stages) { return ((2 * stages + 2) * 8 + 127) / 128 * 128; }

// attention merge scratch: 3 x [pieces <= grid] floats in the record area
constexpr int kMaxGrid = 256;
constexpr int kAttnMergeFloats = 3 * kMaxGrid;

// shared-memory map of one CTA
struct Smem {
    char* ring;        // [stages][kChunkBytes]
    uint64_t* full;    // [stages]
    uint64_t* empty;   // [stages]
    uint64_t* xbar;
    uint64_t* abar;    // attention pairs: the peer's merged half landed (rank 0 of a pair)
    void* x;           // staged input planes
    float* rec;        // [rec_chunks][16][B] / attention scratch
    float* misc;       // 256 floats
    MkPhase* desc;     // [2] phase descriptors (double-buffered bulk copies)
    uint64_t* dbar;    // [2]
    void* gsh;         // GemvShared
    MkChunk* meta;     // [stages] record of the chunk in each ring slot
    int* pstart;       // [nph + 1] this CTA's first chunk record of each phase of the launch
    int* ptiles;       // [nph] first | last << 16 output tile of the CTA's range (-1: none)
};

// Per-phase shared state of a GEMV phase (computed once, read by all warps).
struct GemvShared {
    MkSplit sp;
    int ulo, uhi, Tf;
    unsigned cnt[kMkMaxLocalTiles];  // chunk completions per local tile (0x10000 = tile complete)
    float inv[4];
    unsigned next;                   // dynamic chunk assignment
    unsigned ready;                  // warps that published their finalize operands
    int xpf_ok;                      // xpf holds the residual rows of this CTA's tiles
    int nchunks;                     // this CTA's chunks in the phase
    unsigned released[kMkMaxStages]; // rounds of each ring slot consumed so far (whole launch)
    int pos;                         // length register, read once per launch
    float2 rope[64];                 // kOutQKV: (cos, sin) of position pos
    float xpf[8 * kTileRows * 4];    // kOutResid: residual rows of the CTA's tiles (<= 8 tiles)
    float gpf[8 * kTileRows];        // kOutResid: the next RMSNorm's gamma at those rows
};

// ---------------------------------------------------------------- GEMV ----
template <typename W, int B>
__device__ __forceinline__ void finalize_rows(const MkGemv& g, const GemvShared& sh, int T, int i,
                                              const float (&v)[2][B], const float* inv) {
    using IO = PlaneIO<W>;
    const MkSplit& sp = sh.sp;
    // segment and row of output tile T
    int s = 0;
    if (!sp.dual)
        while (s + 1 < sp.nseg && T >= sp.tbase[s + 1]) ++s;
    const int row = (T - sp.tbase[s]) * kTileRows + i;
    const bool valid = i < kTileRows && row < g.seg[s].rows;  // lanes 16..31 carry no row
    switch (g.out_kind) {
        case kOutPlanes:
            if (valid)
#pragma unroll
                for (int b = 0; b < B; ++b) IO::put(g.out, b, g.out_off[s] + row, v[0][b] * inv[b]);
            break;
        case kOutResid:
            if (valid)
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    float* xr = g.xres + static_cast<size_t>(b) * g.xres_ld + row;
                    const int pr = row - sh.Tf * kTileRows;  // prefetched residual rows of this CTA
                    const float x0 = sh.xpf_ok ? sh.xpf[pr * B + b] : __ldcg(xr);
                    const float x = x0 + v[0][b];
                    *xr = x;
                    IO::put(g.out, b, row, x * (sh.xpf_ok ? sh.gpf[pr] : g.gamma[row]));
                }
            break;
        case kOutSilu:
            if (valid)
#pragma unroll
                for (int b = 0; b < B; ++b) IO::put(g.out, b, row, silu_mul(v[1][b], v[0][b]));
            break;
        case kOutLogits: {
            // all 32 lanes take part in the tile-best reduction (lanes >= 16 carry nothing)
#pragma unroll
            for (int b = 0; b < B; ++b) {
                float bv = -CUDART_INF_F;
                int bi = 0x7fffffff;
                if (valid) {
                    const float x = v[0][b] * inv[b];
                    g.logits[static_cast<size_t>(b) * g.vocab + row] = x;
                    bv = x;
                    bi = row;
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
                if (i == 0) {
                    g.cand_v[T * B + b] = bv;
                    g.cand_i[T * B + b] = bi;
                }
            }
            break;
        }
        default: {  // kOutQKV: segment 0 q, 1 k, 2 v
            const int pos = sh.pos;
            float o[B];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const float x = v[0][b];
                const float y = __shfl_xor_sync(0xffffffffu, x, 1);  // pair partner (rows 2i, 2i+1)
                o[b] = x;
                if (s < 2) {
                    const int e = row % g.d_head;
                    const float2 cs = sh.rope[e >> 1];
                    const float x0 = (e & 1) ? y : x, x1 = (e & 1) ? x : y;
                    o[b] = (e & 1) ? __fadd_rn(__fmul_rn(x0, cs.y), __fmul_rn(x1, cs.x))
                                   : __fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y));
                }
            }
            if (valid) {
                const int h = row / g.d_head, e = row % g.d_head;
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    if (s == 0) {
                        g.qbuf[static_cast<size_t>(b) * g.q_ld + row] = o[b];
                    } else {
                        W* c = static_cast<W*>(s == 1 ? g.kcache : g.vcache);
                        c[b * g.cache_bstride + h * g.cache_hstride + static_cast<long long>(pos) * g.d_head + e] =
                            from_f32<W>(o[b]);
                    }
                }
            }
            break;
        }
    }
}

// Shared-tile exchange of output tile T. The CTA owning T's first unit
// (slot 0) finalizes: it waits for the other contributors' partials (their
// publish is a release-increment of the tile counter, no round trip for
// them) and sums slots 1.. onto its own partial in CTA order. Boundary tiles
// are reduced first in every CTA (ChunkSeq), so the wait is normally one
// poll. Returns false if another CTA finalizes T.
template <int B>
__device__ __forceinline__ bool exchange_pieces(const MkGemv& g, const MkSplit& sp, int T, int cta, int G, int lane,
                                                float (&v)[2][B]) {
    int ta, te;
    sp.tile_span(T, ta, te);
    const int c0 = sp.cta_of(ta, G), c1 = sp.cta_of(te - 1, G);
    if (c0 == c1) return true;  // this CTA covers the whole tile
    // contributors = non-empty CTAs in [c0, c1]: lane l tests CTA base + l
    int np = 0, slot = 0;
    for (int base = c0; base <= c1; base += 32) {
        const int c = base + lane;
        const bool ne = c <= c1 && sp.lo(c + 1, G) > sp.lo(c, G);
        np += __popc(__ballot_sync(0xffffffffu, ne));
        slot += __popc(__ballot_sync(0xffffffffu, ne && c < cta));
    }
    const int subs = sp.subs();
    float* pc = g.pieces + static_cast<size_t>(T) * g.max_pieces * 2 * kTileRows * B;
    // gather the 16 x subs x B partials to lane 0, which publishes them (its
    // own stores + a release increment: no fence by the other lanes)
    float all[2][kTileRows][B];
#pragma unroll
    for (int sb = 0; sb < 2; ++sb)
#pragma unroll
        for (int r = 0; r < kTileRows; ++r)
#pragma unroll
            for (int b = 0; b < B; ++b) all[sb][r][b] = __shfl_sync(0xffffffffu, v[sb][b], r);
    if (slot > 0) {
        if (lane == 0) {
            float4* dst = reinterpret_cast<float4*>(pc + static_cast<size_t>(slot) * 2 * kTileRows * B);
            const float* src = &all[0][0][0];
#pragma unroll
            for (int q = 0; q < 2 * kTileRows * B / 4; ++q)
                dst[q] = make_float4(src[4 * q], src[4 * q + 1], src[4 * q + 2], src[4 * q + 3]);
            red_release_add(g.count + T, 1u);
        }
        return false;
    }
    // slot 0: wait for the np - 1 others, then sum in CTA order
    if (lane == 0)
        while (ld_acquire(g.count + T) < static_cast<unsigned>(np - 1)) {
        }
    __syncwarp();
    fence_acq_rel_gpu();
#pragma unroll
    for (int sb = 0; sb < 2; ++sb)
#pragma unroll
        for (int b = 0; b < B; ++b) {
            float acc = v[sb][b];
            if (lane < kTileRows && sb < subs)
                for (int q = 1; q < np; ++q) acc += __ldcg(pc + ((q * 2 + sb) * kTileRows + lane) * B + b);
            v[sb][b] = acc;
        }
    if (lane == 0) g.count[T] = 0u;
    return true;
}

template <typename W, int B>
__device__ void gemv_phase(const MkGemv& g, const Smem& sm, GemvShared& sh, int tid, int cta, int G, uint32_t& cseq,
                           uint32_t& xphase, int stages, unsigned long long* tr, unsigned long long* ctr, int chunk_lo,
                           int chunk_hi, int tinfo, volatile int* prog) {
    constexpr int ES = sizeof(W);
    const int warp = tid >> 5, lane = tid & 31;
    // ---- stage the input planes (one bulk copy); the finalize operands (RMSNorm
    // sum of squares, RoPE row, residual rows) load in the shadow of that copy ----
    const int Tf = tinfo >= 0 ? (tinfo & 0xFFFF) : 0, Tl = tinfo >= 0 ? (tinfo >> 16) : -1;
    if (tid == 0) {  // (the input planes' bulk copy was issued by the main loop right after the barrier)
        sh.sp.init(g.seg, g.nseg, g.dual, ES, g.exact_split);
        sh.Tf = Tf;
        sh.xpf_ok = g.out_kind == kOutResid && Tl >= Tf && (Tl - Tf + 1) * kTileRows <= 8 * kTileRows;
        sh.next = 0u;
        sh.nchunks = chunk_hi - chunk_lo;
        sh.ready = 0u;
    }
    if (tid < kMkMaxLocalTiles) sh.cnt[tid] = 0u;
    const int rec_per_tile = (g.rec_c0 + g.rec_c1) * kTileRows * B;
    {
        float4* r4 = reinterpret_cast<float4*>(sm.rec);
        const int n4 = g.rec_ntl * rec_per_tile / 4;
        for (int q = tid; q < n4; q += kConsumerThreads) r4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    consumer_sync();
    if (g.out_kind == kOutQKV && tid == kConsumerThreads - 32) {  // (off tid 0's staging path)
        // warm L2 with the K/V rows this CTA reads in the attention phase that
        // follows (rows < pos are final; row pos is appended by this phase)
        const int H = g.seg[0].rows / g.d_head, len = sh.pos + 1;
        const RowSplit rs{B * H * len};
        int r0 = rs.lo(cta, G), r1 = rs.lo(cta + 1, G);
        if (g.attn_pairs) {  // this CTA's half of head cta / 2 (attn_pair_phase)
            const int bh = cta >> 1, hf = cta & 1;
            r0 = r1 = 0;
            if (bh < B * H) {
                r0 = bh * len + len * hf / 2;
                r1 = bh * len + len * (hf + 1) / 2;
            }
        }
        for (int bh = r0 / len; r1 > r0 && bh <= (r1 - 1) / len; ++bh) {
            const int j0 = max(r0 - bh * len, 0), j1 = min(r1 - bh * len, len - 1);
            if (j1 <= j0) continue;
            const long long off = (bh / H) * g.cache_bstride + (bh % H) * g.cache_hstride +
                                  static_cast<long long>(j0) * g.d_head;
            const uint32_t bytes = static_cast<uint32_t>(j1 - j0) * g.d_head * ES;
            for (uint32_t o = 0; o < bytes; o += 16384u) {
                const uint32_t n = min(16384u, bytes - o);
                prefetch_l2_bulk(static_cast<const char*>(g.kcache) + off * ES + o, n);
                prefetch_l2_bulk(static_cast<const char*>(g.vcache) + off * ES + o, n);
            }
        }
    }

    // issue the operand loads (registers), consumed after the x copy lands
    float2 rope_v = make_float2(0.f, 0.f);
    const bool has_rope = g.out_kind == kOutQKV && tid < g.d_head / 2;
    if (has_rope) rope_v = g.rope[static_cast<long long>(sh.pos) * (g.d_head / 2) + tid];
    const int nr = (Tl - Tf + 1) * kTileRows;
    const bool has_xpf = g.out_kind == kOutResid && Tl >= Tf && nr <= 8 * kTileRows;
    float xpf_v[2] = {0.f, 0.f}, gpf_v = 0.f;
    if (has_xpf && tid < nr) {
        const int row = Tf * kTileRows + tid;
        gpf_v = row < g.seg[0].rows ? __ldg(g.gamma + row) : 0.f;
    }
    if (has_xpf)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int q = tid + u * kConsumerThreads;
            if (q < nr * B) {
                const int b = q / nr, r = q - b * nr, row = Tf * kTileRows + r;
                xpf_v[u] = row < g.seg[0].rows ? __ldcg(g.xres + static_cast<size_t>(b) * g.xres_ld + row) : 0.f;
            }
        }
    float ss[B];
#pragma unroll
    for (int b = 0; b < B; ++b) ss[b] = 0.f;
    if (g.norm_src)
#pragma unroll
        for (int b = 0; b < B; ++b) {
            // all of this thread's loads in flight at once (d <= 8 x 1024)
            constexpr int kMaxIt = 8;
            float4 xv[kMaxIt];
#pragma unroll
            for (int it = 0; it < kMaxIt; ++it) {
                const int j = tid * 4 + it * kConsumerThreads * 4;
                xv[it] = j < g.norm_len
                             ? __ldcg(reinterpret_cast<const float4*>(g.norm_src + static_cast<size_t>(b) * g.norm_ld + j))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int it = 0; it < kMaxIt; ++it) {
                ss[b] = fmaf(xv[it].x, xv[it].x, ss[b]);
                ss[b] = fmaf(xv[it].y, xv[it].y, ss[b]);
                ss[b] = fmaf(xv[it].z, xv[it].z, ss[b]);
                ss[b] = fmaf(xv[it].w, xv[it].w, ss[b]);
            }
        }
    const MkSplit& sp = sh.sp;
    if (prog && tid == 0) prog[1] = 10;
    mbar_wait(sm.xbar, xphase & 1u);
    if (prog && tid == 0) prog[1] = 11;
    ++xphase;
    if (tr && tid == 0) tr[1] = gtimer();
    // publish the operands; finalizers wait for all 8 warps (sh.ready) before use
    if (has_rope) sh.rope[tid] = rope_v;
    if (has_xpf && tid < nr) sh.gpf[tid] = gpf_v;
    if (has_xpf)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int q = tid + u * kConsumerThreads;
            if (q < nr * B) {
                const int b = q / nr, r = q - b * nr;
                sh.xpf[r * B + b] = xpf_v[u];
            }
        }
#pragma unroll
    for (int b = 0; b < B; ++b) ss[b] = warp_sum(ss[b]);
    if (lane == 0) {
#pragma unroll
        for (int b = 0; b < B; ++b) sm.misc[warp * 4 + b] = ss[b];
    }
    __syncwarp();
    __threadfence_block();
    if (lane == 0) atomicAdd(&sh.ready, 1u);
    float inv[B];
    bool have_inv = false;
    auto get_inv = [&]() {
        if (have_inv) return;
        if (lane == 0)
            while (*reinterpret_cast<volatile unsigned*>(&sh.ready) < static_cast<unsigned>(kConsumerWarps)) {
            }
        __syncwarp();
        __threadfence_block();
#pragma unroll
        for (int b = 0; b < B; ++b) {
            if (g.norm_src) {
                float t = 0.f;
                for (int w = 0; w < kConsumerWarps; ++w) t += *reinterpret_cast<volatile float*>(&sm.misc[w * 4 + b]);
                inv[b] = 1.0f / sqrtf(t / static_cast<float>(g.norm_len) + g.eps);
            } else {
                inv[b] = 1.f;
            }
        }
        have_inv = true;
    };

    // ---- chunks (boundary tiles first): chunk -> warp cseq % 8; the warp that
    // completes a tile's last chunk finalizes the tile right away ----
    const W* xs = static_cast<const W*>(sm.x);
    const int c_stride[2] = {0, g.rec_c0};
    const uint32_t cbase = cseq;
    const int nchunks = sh.nchunks;
    const uint4* meta = reinterpret_cast<const uint4*>(sm.meta);
    for (;;) {
        // grab the next chunk (dynamic: a warp held up never stalls the ring)
        int jn = 0;
        if (lane == 0) jn = static_cast<int>(atomicAdd(&sh.next, 1u));
        jn = __shfl_sync(0xffffffffu, jn, 0);
        if (jn >= nchunks) break;
        const uint32_t cs = cbase + static_cast<uint32_t>(jn);
        const uint32_t slot = cs % stages, round = cs / stages, par = round & 1u;
        if (prog && lane == 0) { prog[2 + warp] = 100000000 + static_cast<int>(cs); prog[10] = static_cast<int>(cbase); prog[11] = nchunks; }
        // Chunks are grabbed dynamically, so two warps may want the same slot
        // for consecutive rounds; the parity wait can only tell the current
        // round from the previous one. Wait until the slot's previous round
        // is consumed first, then the parity is unambiguous.
        if (lane == 0)
            while (*reinterpret_cast<volatile unsigned*>(&sh.released[slot]) != round) {
            }
        __syncwarp();
        mbar_wait(&sm.full[slot], par);
        if (prog && lane == 0) prog[2 + warp] = 200000000 + static_cast<int>(cs);
        const unsigned long long t_wait = ctr ? gtimer() : 0ull;
        const uint4 mr = meta[slot];
        const MkChunk& ch = *reinterpret_cast<const MkChunk*>(&mr);
        const int nl = ch.nl & 0xF, sub = (ch.nl >> 4) & 1, T = ch.T, k = ch.k, c = ch.c, c_tile = ch.ctile;
        const bool last_of_tile = (ch.nl & 0x20) != 0;
        const int kbase = ch.kbase;
        float* rec = sm.rec + k * rec_per_tile + (c_stride[sub] + c) * kTileRows * B;
        ChunkDot<W, B>::run(sm.ring + static_cast<size_t>(slot) * kChunkBytes, nl, xs, g.in.len, kbase, lane, rec);
        __syncwarp();
        if (ctr && lane == 0 && cs < 8192) {
            ctr[cs * 4 + 1] = t_wait;
            ctr[cs * 4 + 2] = gtimer();
            ctr[cs * 4 + 3] = warp;
        }
        unsigned done = 0;
        if (lane == 0) {
            *reinterpret_cast<volatile unsigned*>(&sh.released[slot]) = round + 1u;
            mbar_arrive(&sm.empty[slot]);
            __threadfence_block();
            // every chunk adds 1; the tile's last chunk adds 0x10000 - c_tile, so the
            // counter reaches exactly 0x10000 when all of the tile's chunks are reduced
            const unsigned add = last_of_tile ? 0x10000u - static_cast<unsigned>(c_tile) : 1u;
            done = atomicAdd(&sh.cnt[k], add) + add == 0x10000u;
        }
        done = __shfl_sync(0xffffffffu, done, 0);
        if (!done) continue;
        __threadfence_block();
        // ---- finalize tile T: sum its chunk records in chunk order ----
        float v[2][B];
        const float* rt = sm.rec + k * rec_per_tile;
#pragma unroll
        for (int sb = 0; sb < 2; ++sb)
#pragma unroll
            for (int b = 0; b < B; ++b) {
                float acc = 0.f;
                if (lane < kTileRows) {
                    const int n = sb ? g.rec_c1 : g.rec_c0;
                    for (int q = 0; q < n; ++q) acc += rt[((c_stride[sb] + q) * kTileRows + lane) * B + b];
                }
                v[sb][b] = acc;
            }
        // tile-aligned ranges: one owner per tile; even splits: a shared tile is
        // finalized by the CTA holding its first unit after the others' pieces
        if (g.exact_split && !exchange_pieces<B>(g, sp, T, cta, G, lane, v)) continue;
        get_inv();
        finalize_rows<W, B>(g, sh, T, lane, v, inv);
    }
    if (prog && lane == 0) prog[2 + warp] = 3000000 + nchunks;
    cseq = cbase + static_cast<uint32_t>(nchunks);
    consumer_sync();
    if (tr && tid == 0) tr[3] = gtimer();
}

// ----------------------------------------------------------- attention ----
template <typename T, int PER>
__device__ __forceinline__ void load_kv_row(const T* p, float* out) {
    if constexpr (sizeof(T) == 2 && PER == 4) {
        const uint2 v = __ldcg(reinterpret_cast<const uint2*>(p));
        out[0] = bf16lo(v.x);
        out[1] = bf16hi(v.x);
        out[2] = bf16lo(v.y);
        out[3] = bf16hi(v.y);
    } else if constexpr (sizeof(T) == 4 && PER == 4) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
        out[0] = v.x;
        out[1] = v.y;
        out[2] = v.z;
        out[3] = v.w;
    } else {
#pragma unroll
        for (int e = 0; e < PER; ++e) out[e] = to_f32<T>(p[e]);
    }
}

// K/V row slice of one lane kept packed while in flight (bf16: 4 values in a uint2)
template <typename E, int PER>
struct KvRaw {
    struct T4 {
        float v[PER];
    };
    using T = T4;
    static __device__ __forceinline__ T4 load(const E* p) {
        T4 r;
        load_kv_row<E, PER>(p, r.v);
        return r;
    }
    static __device__ __forceinline__ void unpack(const T4& r, float* out) {
#pragma unroll
        for (int e = 0; e < PER; ++e) out[e] = r.v[e];
    }
};
template <>
struct KvRaw<__nv_bfloat16, 4> {
    using T = uint2;
    static __device__ __forceinline__ uint2 load(const __nv_bfloat16* p) {
        return __ldcg(reinterpret_cast<const uint2*>(p));
    }
    static __device__ __forceinline__ void unpack(const uint2& v, float* out) {
        out[0] = bf16lo(v.x);
        out[1] = bf16hi(v.x);
        out[2] = bf16lo(v.y);
        out[3] = bf16hi(v.y);
    }
};

// Merge of head bh's warp partials (warps [w0, w1) of this CTA): a head held by
// one CTA is normalized directly into the o-projection's input planes; a head
// shared by several CTAs goes through per-CTA pieces, merged in CTA order by
// the CTA holding its newest keys (the others publish with a release
// increment and never wait).
template <typename W, int B, int DH>
__device__ void attn_merge(const MkAttn& a, const Smem& sm, int tid, int cta, int G, const RowSplit& rs, int len, int bh,
                           int w0, int w1) {
    constexpr int ST = DH + 2;
    float* wst = sm.rec;
    const int b = bh / a.n_heads, h = bh % a.n_heads;
    const int lo_bh = bh * len, hi_bh = lo_bh + len;
    const int c0 = rs.cta_of(lo_bh, G), c1 = rs.cta_of(hi_bh - 1, G);
    const int np = rs.nonempty(c0, c1 + 1, G);
    float M = -CUDART_INF_F;
    for (int w = w0; w < w1; ++w) M = fmaxf(M, wst[w * ST + DH + 1]);
    float* part = a.partial + static_cast<long long>(bh) * a.splits * ST;
    if (np > 1) {
        const int slot = rs.nonempty(c0, cta, G);
        const bool fin = slot == np - 1;
        float* own = fin ? sm.misc + 96 : part + slot * ST;  // (misc[96..226) is free here)
        for (int e = tid; e < DH + 1; e += kConsumerThreads) {
            float t = 0.f;
            for (int w = w0; w < w1; ++w) {
                const float mw = wst[w * ST + DH + 1];
                if (mw != -CUDART_INF_F) t += wst[w * ST + e] * expf(mw - M);
            }
            own[e] = t;
        }
        if (tid == 0) own[DH + 1] = M;
        consumer_sync();
        if (!fin) {
            if (tid == 0) {
                fence_acq_rel_gpu();
                red_release_add(a.count + bh, 1u);
            }
        } else {
            if (tid == 0)
                while (ld_acquire(a.count + bh) < static_cast<unsigned>(np - 1)) {
                }
            consumer_sync();
            // one round of loads: every piece's (m, l, acc[e]) in flight at once,
            // then an online merge in CTA order (running max, rescaled sums)
            if (tid < DH) {
                const int e = tid;
                constexpr int QB = 8;
                float MM = -CUDART_INF_F, L = 0.f, o = 0.f;
                auto fold = [&](float mq, float lq, float aq) {
                    const float mn = fmaxf(MM, mq);
                    const float so = expf(MM - mn), sq = expf(mq - mn);
                    L = fmaf(L, so, lq * sq);
                    o = fmaf(o, so, aq * sq);
                    MM = mn;
                };
                for (int q0 = 0; q0 < np - 1; q0 += QB) {
                    float mv[QB], lv[QB], av[QB];
#pragma unroll
                    for (int u = 0; u < QB; ++u) {
                        const int q = min(q0 + u, np - 2);
                        mv[u] = __ldcg(part + q * ST + DH + 1);
                        lv[u] = __ldcg(part + q * ST + DH);
                        av[u] = __ldcg(part + q * ST + e);
                    }
#pragma unroll
                    for (int u = 0; u < QB; ++u)
                        if (q0 + u < np - 1) fold(mv[u], lv[u], av[u]);
                }
                fold(own[DH + 1], own[DH], own[e]);
                PlaneIO<W>::put(a.out, b, h * DH + e, o / L);
            }
            if (tid == 0) a.count[bh] = 0u;
        }
    } else {
        float L = 0.f;
        for (int w = w0; w < w1; ++w) {
            const float mw = wst[w * ST + DH + 1];
            if (mw != -CUDART_INF_F) L += wst[w * ST + DH] * expf(mw - M);
        }
        const float invL = 1.0f / L;
        for (int e = tid; e < DH; e += kConsumerThreads) {
            float t = 0.f;
            for (int w = w0; w < w1; ++w) {
                const float mw = wst[w * ST + DH + 1];
                if (mw != -CUDART_INF_F) t += wst[w * ST + e] * expf(mw - M);
            }
            PlaneIO<W>::put(a.out, b, h * DH + e, t * invL);
        }
    }
    consumer_sync();
}

// Dense-KV decode attention (online softmax math.hpp:56-101).
// The B*H*len key rows are split evenly over the CTAs. A CTA works on its
// heads two at a time (with B*H < grid it never has more than two), the warps
// split between them in proportion to their rows, so a CTA straddling a head
// boundary takes no longer than one inside a head. Each warp streams its rows
// 16 at a time (all of a batch's K/V loads in flight), then the heads are
// merged, the one shared with the next CTA first (publish, no wait).
template <typename W, int B, int DH>
__device__ void attn_pair_phase(const MkAttn& a, const Smem& sm, int tid, int cta, int pos, uint32_t aidx);

template <typename W, int B, int DH>
__device__ void attn_phase(const MkAttn& a, const Smem& sm, int tid, int cta, int G, int pos, uint32_t aidx) {
    constexpr int PER = DH / 32, KU = 16, ST = DH + 2;
    const int warp = tid >> 5, lane = tid & 31;
    const int len = pos + 1;
    uint32_t ncl = 1;
    if (a.pairs) asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
    if (a.pairs && ncl == 2) {  // (a launch without the cluster attribute, e.g. a profiler's replay, takes the row split)
        attn_pair_phase<W, B, DH>(a, sm, tid, cta, pos, aidx);
        return;
    }
    RowSplit rs{B * a.n_heads * len};
    const int r0 = rs.lo(cta, G), r1 = rs.lo(cta + 1, G);
    if (r1 <= r0) return;
    float* wst = sm.rec;  // [warps][DH + 2]: acc, l, m
    const int bh_first = r0 / len, bh_last = (r1 - 1) / len;
    for (int bh_hi = bh_last; bh_hi >= bh_first; bh_hi -= 2) {
        const int bh_lo = max(bh_first, bh_hi - 1);
        auto span = [&](int bh, int& j0, int& j1) {
            const int lo_bh = bh * len, hi_bh = lo_bh + len;
            j0 = (r0 > lo_bh ? r0 : lo_bh) - lo_bh;
            j1 = (r1 < hi_bh ? r1 : hi_bh) - lo_bh;
        };
        int jl0, jl1, jh0, jh1;
        span(bh_lo, jl0, jl1);
        span(bh_hi, jh0, jh1);
        int w_lo = 0;  // warps [0, w_lo) on bh_lo, [w_lo, 8) on bh_hi
        if (bh_lo != bh_hi) {
            const int nl = jl1 - jl0, nh = jh1 - jh0;
            w_lo = (2 * kConsumerWarps * nl + (nl + nh)) / (2 * (nl + nh));  // round(8 nl / (nl + nh))
            w_lo = min(max(w_lo, 1), kConsumerWarps - 1);
        }
        const bool on_lo = warp < w_lo;
        const int bh = on_lo ? bh_lo : bh_hi;
        const int j0 = on_lo ? jl0 : jh0, j1 = on_lo ? jl1 : jh1;
        const int wi = on_lo ? warp : warp - w_lo, nw = on_lo ? w_lo : kConsumerWarps - w_lo;
        const int b = bh / a.n_heads, h = bh % a.n_heads;
        const W* Kc = static_cast<const W*>(a.kcache) + b * a.cache_bstride + h * a.cache_hstride;
        const W* Vc = static_cast<const W*>(a.vcache) + b * a.cache_bstride + h * a.cache_hstride;
        float qr[PER];
        {
            const float* q = a.qbuf + static_cast<size_t>(b) * a.q_ld + h * DH + lane * PER;
#pragma unroll
            for (int e = 0; e < PER; ++e) qr[e] = __ldcg(q + e) * a.scale;
        }
        const int n = j1 - j0;
        const int k0 = j0 + n * wi / nw, k1 = j0 + n * (wi + 1) / nw;
        float m = -CUDART_INF_F, l = 0.f, acc[PER];
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[e] = 0.f;
        using Raw = typename KvRaw<W, PER>::T;
        for (int kb = k0; kb < k1; kb += KU) {
            Raw kq[KU], vq[KU];
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                const int jj = min(kb + u, k1 - 1);  // clamp: duplicate loads are masked below
                kq[u] = KvRaw<W, PER>::load(Kc + static_cast<long long>(jj) * DH + lane * PER);
                vq[u] = KvRaw<W, PER>::load(Vc + static_cast<long long>(jj) * DH + lane * PER);
            }
            float sc[KU];
            float mb = -CUDART_INF_F;
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                float kr[PER];
                KvRaw<W, PER>::unpack(kq[u], kr);
                float d = 0.f;
#pragma unroll
                for (int e = 0; e < PER; ++e) d = fmaf(qr[e], kr[e], d);
                d = warp_sum(d);
                sc[u] = kb + u < k1 ? d : -CUDART_INF_F;
                mb = fmaxf(mb, sc[u]);
            }
            const float mn = fmaxf(m, mb);
            const float r = expf(m - mn);  // exp(-inf) = 0 on the first round
            l *= r;
#pragma unroll
            for (int e = 0; e < PER; ++e) acc[e] *= r;
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                float vr[PER];
                KvRaw<W, PER>::unpack(vq[u], vr);
                const float w = expf(sc[u] - mn);
                l += w;
#pragma unroll
                for (int e = 0; e < PER; ++e) acc[e] = fmaf(w, vr[e], acc[e]);
            }
            m = mn;
        }
#pragma unroll
        for (int e = 0; e < PER; ++e) wst[warp * ST + lane * PER + e] = acc[e];
        if (lane == 0) {
            wst[warp * ST + DH] = l;
            wst[warp * ST + DH + 1] = m;
        }
        consumer_sync();
        if (bh_lo != bh_hi) {
            attn_merge<W, B, DH>(a, sm, tid, cta, G, rs, len, bh_hi, w_lo, kConsumerWarps);
            attn_merge<W, B, DH>(a, sm, tid, cta, G, rs, len, bh_lo, 0, w_lo);
        } else {
            attn_merge<W, B, DH>(a, sm, tid, cta, G, rs, len, bh_hi, 0, kConsumerWarps);
        }
    }
}

// One CTA pair (a thread-block cluster of 2 on one TPC) per (b, h): CTA half
// hf attends keys [len hf / 2, len (hf + 1) / 2) with its 8 warps (16-key
// batches, online softmax), merges its warps into one piece (acc, l, m), and
// the second CTA stores its piece straight into the first one's shared memory
// (st.shared::cluster + a release arrive per element on the first CTA's
// mbarrier); the first CTA merges the two pieces and writes the o-projection
// input. No global scratch, no cross-CTA polling.
template <typename W, int B, int DH>
__device__ void attn_pair_phase(const MkAttn& a, const Smem& sm, int tid, int cta, int pos, uint32_t aidx) {
    constexpr int PER = DH / 32, KU = 16, ST = DH + 2;
    const int warp = tid >> 5, lane = tid & 31;
    const int len = pos + 1;
    const int bh = cta >> 1, hf = cta & 1;
    if (bh >= B * a.n_heads) return;
    const int b = bh / a.n_heads, h = bh % a.n_heads;
    const int lo = len * hf / 2, hi = len * (hf + 1) / 2;
    const int n = hi - lo;
    const int k0 = lo + n * warp / kConsumerWarps, k1 = lo + n * (warp + 1) / kConsumerWarps;
    const W* Kc = static_cast<const W*>(a.kcache) + b * a.cache_bstride + h * a.cache_hstride;
    const W* Vc = static_cast<const W*>(a.vcache) + b * a.cache_bstride + h * a.cache_hstride;
    float qr[PER];
    {
        const float* q = a.qbuf + static_cast<size_t>(b) * a.q_ld + h * DH + lane * PER;
#pragma unroll
        for (int e = 0; e < PER; ++e) qr[e] = __ldcg(q + e) * a.scale;
    }
    float m = -CUDART_INF_F, l = 0.f, acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.f;
    using Raw = typename KvRaw<W, PER>::T;
    for (int kb = k0; kb < k1; kb += KU) {
        Raw kq[KU], vq[KU];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            const int jj = min(kb + u, k1 - 1);  // clamp: duplicate loads are masked below
            kq[u] = KvRaw<W, PER>::load(Kc + static_cast<long long>(jj) * DH + lane * PER);
            vq[u] = KvRaw<W, PER>::load(Vc + static_cast<long long>(jj) * DH + lane * PER);
        }
        float sc[KU];
        float mb = -CUDART_INF_F;
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            float kr[PER];
            KvRaw<W, PER>::unpack(kq[u], kr);
            float d = 0.f;
#pragma unroll
            for (int e = 0; e < PER; ++e) d = fmaf(qr[e], kr[e], d);
            d = warp_sum(d);
            sc[u] = kb + u < k1 ? d : -CUDART_INF_F;
            mb = fmaxf(mb, sc[u]);
        }
        const float mn = fmaxf(m, mb);
        const float r = expf(m - mn);  // exp(-inf) = 0 on the first round
        l *= r;
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[e] *= r;
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            float vr[PER];
            KvRaw<W, PER>::unpack(vq[u], vr);
            const float w = expf(sc[u] - mn);
            l += w;
#pragma unroll
            for (int e = 0; e < PER; ++e) acc[e] = fmaf(w, vr[e], acc[e]);
        }
        m = mn;
    }
    float* wst = sm.rec;  // [warps][DH + 2]: acc, l, m
#pragma unroll
    for (int e = 0; e < PER; ++e) wst[warp * ST + lane * PER + e] = acc[e];
    if (lane == 0) {
        wst[warp * ST + DH] = l;
        wst[warp * ST + DH + 1] = m;
    }
    consumer_sync();
    // this CTA's piece: element e < DH (acc), DH (l); every thread computes the
    // CTA max M itself (8 values)
    float M = -CUDART_INF_F;
    for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, wst[w * ST + DH + 1]);
    auto piece = [&](int e) {
        float t = 0.f;
        for (int w = 0; w < kConsumerWarps; ++w) {
            const float mw = wst[w * ST + DH + 1];
            if (mw != -CUDART_INF_F) t += wst[w * ST + e] * expf(mw - M);
        }
        return t;
    };
    float* peer = sm.misc;  // [DH + 2] in the pair's first CTA: the second CTA's piece
    if (hf == 1) {
        if (tid < DH + 2) {
            const float v = tid == DH + 1 ? M : piece(tid);
            uint32_t ra, rb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;"
                         : "=r"(ra)
                         : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(peer + tid))));
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;"
                         : "=r"(rb)
                         : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(sm.abar))));
            asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
        }
        consumer_sync();
        return;
    }
    if (tid < DH) {
        const float own = piece(tid), own_l = piece(DH);
        {  // the peer's piece (acquire at cluster scope)
            const uint32_t ba = static_cast<uint32_t>(__cvta_generic_to_shared(sm.abar));
            asm volatile(
                "{\n.reg .pred p;\nAW_%=:\n"
                "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
                "@!p bra AW_%=;\n}\n" ::"r"(ba),
                "r"(aidx & 1u)
                : "memory");
        }
        const float pm = *reinterpret_cast<volatile float*>(peer + DH + 1);
        const float pl = *reinterpret_cast<volatile float*>(peer + DH);
        const float pa = *reinterpret_cast<volatile float*>(peer + tid);
        const float MM = fmaxf(M, pm);
        const float so = M == -CUDART_INF_F ? 0.f : expf(M - MM), sp = pm == -CUDART_INF_F ? 0.f : expf(pm - MM);
        const float L = own_l * so + pl * sp;
        PlaneIO<W>::put(a.out, b, h * DH + tid, (own * so + pa * sp) / L);
    }
    consumer_sync();
}

// ------------------------------------------------------- argmax / vec ----
template <int B>
__device__ void argmax_phase(const MkArgmax& m, const Smem& sm, int tid, int cta) {
    if (cta != 0) return;
    const int warp = tid >> 5, lane = tid & 31;
    float* sv = sm.misc;
    int* si = reinterpret_cast<int*>(sm.misc + 64);
    for (int b = 0; b < B; ++b) {
        float bv = -CUDART_INF_F;
        int bi = 0x7fffffff;
        for (int t = tid; t < m.ntiles; t += kConsumerThreads) {
            const float v = __ldcg(m.cand_v + t * B + b);
            const int i = __ldcg(m.cand_i + t * B + b);
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
            sv[warp * 4 + b] = bv;
            si[warp * 4 + b] = bi;
        }
    }
    consumer_sync();
    if (tid == 0) {
        const int step = m.step ? *m.step : 0;
        for (int b = 0; b < B; ++b) {
            float bv = -CUDART_INF_F;
            int bi = 0x7fffffff;
            for (int w = 0; w < kConsumerWarps; ++w)
                if (better(sv[w * 4 + b], si[w * 4 + b], bv, bi)) {
                    bv = sv[w * 4 + b];
                    bi = si[w * 4 + b];
                }
            if (bi == 0x7fffffff) bi = 0;
            m.tokens[b] = bi;
            if (m.out) m.out[static_cast<long long>(b) * m.out_ld + step] = bi;
        }
        *m.pos += m.pos_inc;
        if (m.step) *m.step = step + 1;
    }
}

template <typename W, int B>
__device__ void vec_phase(const MkVec& v, int tid, int cta, int G) {
    const int i0 = static_cast<int>(static_cast<long long>(v.len) * cta / G);
    const int i1 = static_cast<int>(static_cast<long long>(v.len) * (cta + 1) / G);
#pragma unroll
    for (int b = 0; b < B; ++b) {
        const W* er = v.emb ? static_cast<const W*>(v.emb) + static_cast<long long>(__ldcg(v.tokens + b)) * v.emb_ld
                            : nullptr;
        for (int i = i0 + tid; i < i1; i += kConsumerThreads) {
            const float x = er ? to_f32<W>(er[i]) : __ldcg(v.src + static_cast<size_t>(b) * v.src_ld + i);
            if (v.xres) v.xres[static_cast<size_t>(b) * v.xres_ld + i] = x;
            PlaneIO<W>::put(v.out, b, i, x * v.gamma[i]);
        }
    }
}

// ----------------------------------------------------------- the kernel --
template <typename W, int B, int DH>
__global__ void __launch_bounds__(kThreads, 1) decode_mk_kernel(const __grid_constant__ MkLaunch L) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem sm;
    sm.ring = reinterpret_cast<char*>(smem_raw);
    sm.full = reinterpret_cast<uint64_t*>(smem_raw + static_cast<size_t>(L.stages) * kChunkBytes);
    sm.empty = sm.full + L.stages;
    sm.xbar = sm.empty + L.stages;
    sm.abar = sm.xbar + 1;
    sm.x = reinterpret_cast<char*>(sm.full) + mk_barrier_bytes(L.stages);
    sm.rec = reinterpret_cast<float*>(static_cast<char*>(sm.x) + L.x_bytes);
    const int rec_floats = std::max({L.rec_chunks * kTileRows * B, kConsumerWarps * (DH + 2), kAttnMergeFloats});
    sm.misc = sm.rec + rec_floats;
    sm.desc = reinterpret_cast<MkPhase*>(sm.misc + 256);
    sm.dbar = reinterpret_cast<uint64_t*>(sm.desc + 2);
    sm.gsh = sm.dbar + 2;
    sm.meta = reinterpret_cast<MkChunk*>(static_cast<char*>(sm.gsh) + (sizeof(GemvShared) + 15) / 16 * 16);
    sm.pstart = reinterpret_cast<int*>(sm.meta + L.stages);
    sm.ptiles = sm.pstart + (L.p_end - L.p_begin + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, cta = blockIdx.x, G = gridDim.x;
    if (tid == 0) {
        for (int i = 0; i < L.stages; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        mbar_init(sm.xbar, 1);
        mbar_init(sm.abar, DH + 2);  // the peer's DH + 2 remote stores, one release arrive each
        mbar_init(&sm.dbar[0], 1);
        mbar_init(&sm.dbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kConsumerWarps) {
        // ================= producer: weight stream of every GEMV phase =================
        // Walks this CTA's precomputed chunk records (host-built, in the
        // consumers' order), 32 at a time: lane i loads record i of the batch,
        // lane 0 issues them; the only wait is for a free ring slot.
        const uint64_t policy = evict_first_policy();
        const int* st = L.chunk_start + static_cast<size_t>(cta) * (L.nphases + 1);
        const int i0 = st[L.p_begin], i1 = st[L.p_end];
        if (L.progress && lane == 0) {
            L.progress[cta * 16 + 14] = i0;
            L.progress[cta * 16 + 15] = i1;
        }
        uint4* meta = reinterpret_cast<uint4*>(sm.meta);
        uint32_t seq = 0;
        for (int rep = 0; rep < (L.reps > 1 ? L.reps : 1); ++rep)
        for (int ib = i0; ib < i1; ib += 32) {
            uint4 rec = make_uint4(0u, 0u, 0u, 0u);
            if (ib + lane < i1) rec = __ldg(reinterpret_cast<const uint4*>(L.chunks + ib + lane));
            // L2 prefetch L.l2_ahead chunks beyond the one being issued: HBM keeps
            // streaming while the ring is full (grid barrier, input staging)
            uint4 ahd = make_uint4(0u, 0u, 0u, 0u);
            if (L.l2_ahead > 0 && ib + L.l2_ahead + lane < i1)
                ahd = __ldg(reinterpret_cast<const uint4*>(L.chunks + ib + L.l2_ahead + lane));
            const int n = min(32, i1 - ib);
            for (int q = 0; q < n; ++q, ++seq) {
                uint4 r, a;
                r.x = __shfl_sync(0xffffffffu, rec.x, q);
                r.y = __shfl_sync(0xffffffffu, rec.y, q);
                r.z = __shfl_sync(0xffffffffu, rec.z, q);
                r.w = __shfl_sync(0xffffffffu, rec.w, q);
                a.x = __shfl_sync(0xffffffffu, ahd.x, q);
                a.y = __shfl_sync(0xffffffffu, ahd.y, q);
                a.w = __shfl_sync(0xffffffffu, ahd.w, q);
                if (lane == 0) {
                    if (a.x | a.y) {
                        const MkChunk& ah = *reinterpret_cast<const MkChunk*>(&a);
                        prefetch_l2_bulk(ah.src, static_cast<uint32_t>(ah.nl & 0xF) * kLineTileBytes);
                    }
                    const MkChunk& ch = *reinterpret_cast<const MkChunk*>(&r);
                    const uint32_t slot = seq % L.stages;
                    const uint32_t bytes = static_cast<uint32_t>(ch.nl & 0xF) * kLineTileBytes;
                    if (L.progress) L.progress[cta * 16 + 12] = static_cast<int>(seq);
                    mbar_wait(&sm.empty[slot], ((seq / L.stages) & 1u) ^ 1u);
                    if (L.progress) L.progress[cta * 16 + 13] = static_cast<int>(seq);
                    meta[slot] = r;
                    mbar_expect_tx(&sm.full[slot], bytes);
                    bulk_g2s(sm.ring + static_cast<size_t>(slot) * kChunkBytes, ch.src, bytes, &sm.full[slot], policy);
                    if (L.trace && cta == 0 && seq < 8192)
                        L.trace[static_cast<size_t>(G) * (L.p_end - L.p_begin) * 16 + seq * 4] = gtimer();
                }
                __syncwarp();
            }
        }
        return;
    }

    // ================= consumers =================
    constexpr uint32_t kDescBytes = sizeof(MkPhase);
    if (tid == 0) {  // descriptor of the first phase
        mbar_expect_tx(&sm.dbar[0], kDescBytes);
        bulk_g2s_plain(&sm.desc[0], &L.phases[L.p_begin], kDescBytes, &sm.dbar[0]);
    }
    GemvShared& gsh = *static_cast<GemvShared*>(sm.gsh);
    if (tid < kMkMaxStages) gsh.released[tid] = 0u;
    {  // this CTA's rows of the chunk tables, once per launch
        const int* cs = L.chunk_start + static_cast<size_t>(cta) * (L.nphases + 1) + L.p_begin;
        const int* ct = L.chunk_tiles + static_cast<size_t>(cta) * L.nphases + L.p_begin;
        for (int i = tid; i <= L.p_end - L.p_begin; i += kConsumerThreads) {
            sm.pstart[i] = __ldg(cs + i);
            if (i < L.p_end - L.p_begin) sm.ptiles[i] = __ldg(ct + i);
        }
    }
    if (tid == 0) gsh.pos = L.pos ? __ldcg(L.pos) : 0;  // constant until the argmax phase (last of a step)
    consumer_sync();
    uint32_t cseq = 0, xphase = 0, aidx = 0;
    const int nph = L.p_end - L.p_begin;
    // reps > 1: the phase program runs reps times back to back (reps decode steps
    // in one launch); gi counts phases over the whole launch
    const int reps = L.reps > 1 ? L.reps : 1, ntot = nph * reps;
    for (int gi = 0; gi < ntot; ++gi) {
        const int idx = gi % nph, p = L.p_begin + idx, buf = gi & 1;
        unsigned long long* tr = L.trace ? L.trace + (static_cast<size_t>(cta) * nph + idx) * 16 : nullptr;
        if (L.progress && tid == 0) {
            L.progress[cta * 16] = p;
            L.progress[cta * 16 + 1] = 0;
        }
        if (tid == 0) {
            if (gi > 0) {  // grid barrier: every CTA finished phase gi-1
                const unsigned target = static_cast<unsigned>(gi) * G;
                while (ld_acquire(L.bar) < target) {
                }
                if (idx == 0) gsh.pos = L.pos ? __ldcg(L.pos) : 0;  // next step: the argmax phase advanced it
            }
            // a GEMV phase's input planes: one bulk copy issued the moment the
            // barrier passes (sm.x's readers finished with the previous phase)
            mbar_wait(&sm.dbar[buf], (gi >> 1) & 1u);
            const MkPhase& nx = sm.desc[buf];
            if (nx.kind == kMkGemv) {
                const uint32_t xbytes = static_cast<uint32_t>(B) * nx.g.in.len * PlaneIO<W>::kBytesPerElem;
                fence_proxy_async_global();
                mbar_expect_tx(sm.xbar, xbytes);
                bulk_g2s_plain(sm.x, nx.g.in.p, xbytes, sm.xbar);
            }
        }
        consumer_sync();
        if (tid == 0 && gi + 1 < ntot) {  // prefetch the next descriptor (its buffer's readers are done)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&sm.dbar[buf ^ 1], kDescBytes);
            bulk_g2s_plain(&sm.desc[buf ^ 1], &L.phases[L.p_begin + (gi + 1) % nph], kDescBytes, &sm.dbar[buf ^ 1]);
        }
        if (tr && tid == 0) for (int q = 0; q < 16; ++q) if (q != 5 && q != 6) tr[q] = gtimer();
        if (L.progress && tid == 0) L.progress[cta * 16 + 1] = 1;
        mbar_wait(&sm.dbar[buf], (gi >> 1) & 1u);
        if (L.progress && tid == 0) L.progress[cta * 16 + 1] = 2;
        const MkPhase& ph = sm.desc[buf];
        switch (ph.kind) {
            case kMkGemv: gemv_phase<W, B>(ph.g, sm, gsh, tid, cta, G, cseq, xphase, L.stages, tr, tr && cta == 0 ? L.trace + static_cast<size_t>(G) * nph * 16 : nullptr, sm.pstart[idx], sm.pstart[idx + 1], sm.ptiles[idx], L.progress ? L.progress + cta * 16 : nullptr); break;
            case kMkAttn: attn_phase<W, B, DH>(ph.a, sm, tid, cta, G, gsh.pos, aidx++); break;
            case kMkArgmax: argmax_phase<B>(ph.m, sm, tid, cta); break;
            default: vec_phase<W, B>(ph.v, tid, cta, G); break;
        }
        if (L.progress && tid == 0) L.progress[cta * 16 + 1] = 3;
        consumer_sync();
        if (L.progress && tid == 0) L.progress[cta * 16 + 1] = 4;
        if (tr && tid == 0) tr[4] = gtimer();
        if (tid == 0) {  // arrive (release): this CTA's writes of phase gi are complete
            if (gi + 1 < ntot) {
                red_release_add(L.bar, 1u);  // fire and forget
            } else {
                const unsigned v = atom_add_acq_rel(L.bar, 1u) + 1u;
                if (v == static_cast<unsigned>(ntot) * G) *L.bar = 0u;  // last arrival of the launch: reset
            }
        }
    }
}

template <typename W, int B, int DH>
void launch_t(const MkLaunch& L, cudaStream_t s) {
    auto fn = decode_mk_kernel<W, B, DH>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem_bytes);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(L.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = L.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = L.cluster2 ? 2 : 1;
    cudaLaunchKernelEx(&cfg, fn, L);
}

}  // namespace mk

// --------------------------------------------------------- host mirrors --
int mk_units(const GemvSeg* seg, int nseg, int dual, int esize) {
    MkSplit sp;
    sp.init(seg, nseg, dual, esize);
    return sp.total;
}

int mk_out_tiles(const GemvSeg* seg, int nseg, int dual, int esize) {
    MkSplit sp;
    sp.init(seg, nseg, dual, esize);
    return sp.out_tiles;
}

void mk_split_stats(const GemvSeg* seg, int nseg, int dual, int esize, int grid, int exact, int* max_pieces,
                    int* rec_ntl, int* rec_c0, int* rec_c1) {
    MkSplit sp;
    sp.init(seg, nseg, dual, esize, exact);
    int mp = 1;
    for (int T = 0; T < sp.out_tiles; ++T) {
        int a, e;
        sp.tile_span(T, a, e);
        mp = std::max(mp, sp.nonempty(sp.cta_of(a, grid), sp.cta_of(e - 1, grid) + 1, grid));
    }
    int ntl = 1;
    for (int c = 0; c < grid; ++c) {
        const int ulo = sp.lo(c, grid), uhi = sp.lo(c + 1, grid);
        if (ulo < uhi) ntl = std::max(ntl, sp.tile_of(uhi - 1) - sp.tile_of(ulo) + 1);
    }
    int c0 = 0, c1 = 0;
    if (dual) {
        c0 = (sp.nlines[0] + kChunkLines - 1) / kChunkLines;
        c1 = (sp.nlines[1] + kChunkLines - 1) / kChunkLines;
    } else {
        for (int s = 0; s < nseg; ++s) c0 = std::max(c0, (sp.nlines[s] + kChunkLines - 1) / kChunkLines);
    }
    *max_pieces = mp;
    *rec_ntl = ntl;
    *rec_c0 = c0;
    *rec_c1 = c1;
}

void mk_build_chunks(const MkPhase* phases, int nphases, int grid, int esize, std::vector<MkChunk>& out,
                     std::vector<int>& start, std::vector<int>& tiles) {
    out.clear();
    start.assign(static_cast<size_t>(grid) * (nphases + 1), 0);
    tiles.assign(static_cast<size_t>(grid) * nphases, -1);
    for (int c = 0; c < grid; ++c) {
        for (int p = 0; p < nphases; ++p) {
            start[static_cast<size_t>(c) * (nphases + 1) + p] = static_cast<int>(out.size());
            if (phases[p].kind != kMkGemv) continue;
            const MkGemv& g = phases[p].g;
            MkSplit sp;
            sp.init(g.seg, g.nseg, g.dual, esize, g.exact_split);
            const int ulo = sp.lo(c, grid), uhi = sp.lo(c + 1, grid);
            if (ulo >= uhi) continue;
            const int Tf = sp.tile_of(ulo);
            tiles[static_cast<size_t>(c) * nphases + p] = Tf | (sp.tile_of(uhi - 1) << 16);
            ChunkSeq cs;
            cs.begin(sp, ulo, uhi);
            int T_prev = -1, ctile = 0;
            const size_t first = out.size();
            while (!cs.done()) {
                MkChunk ch{};
                const int nl = cs.it.lines(sp), s = cs.it.s;
                const int T = cs.tile(sp);
                ctile = T == T_prev ? ctile + 1 : 0;
                T_prev = T;
                const WLayout lay = g.seg[s].layout(esize);
                ch.src = static_cast<const char*>(g.seg[s].w) + static_cast<size_t>(cs.it.t) * lay.tile_bytes() +
                         static_cast<size_t>(cs.it.line) * kLineTileBytes;
                const int kbase = g.seg[s].x_off + cs.it.line * (kLineBytes / esize);
                if (T > 0xFFFF || kbase > 0xFFFF || T - Tf > 255 || cs.c_run > 255 || ctile > 255)
                    throw std::runtime_error("decode megakernel: chunk record field overflow");
                ch.T = static_cast<uint16_t>(T);
                ch.kbase = static_cast<uint16_t>(kbase);
                ch.nl = static_cast<uint8_t>(nl | (cs.sub(sp) ? 0x10 : 0));
                ch.k = static_cast<uint8_t>(T - Tf);
                ch.c = static_cast<uint8_t>(cs.c_run);
                ch.ctile = static_cast<uint8_t>(ctile);
                cs.advance(sp, nl);
                out.push_back(ch);
            }
            // mark the last chunk of every output tile
            for (size_t i = first; i < out.size(); ++i)
                if (i + 1 == out.size() || out[i + 1].T != out[i].T) out[i].nl |= 0x20;
        }
        start[static_cast<size_t>(c) * (nphases + 1) + nphases] = static_cast<int>(out.size());
    }
}

static int rec_floats(int rec_chunks, int batch, int d_head) {
    return std::max({rec_chunks * kTileRows * batch, mk::kConsumerWarps * (d_head + 2), mk::kAttnMergeFloats});
}

int mk_smem_bytes(int stages, int x_bytes, int rec_chunks, int batch, int d_head, int nphases) {
    return stages * kChunkBytes + mk::mk_barrier_bytes(stages) + x_bytes + rec_floats(rec_chunks, batch, d_head) * 4 +
           256 * 4 + 2 * static_cast<int>(sizeof(MkPhase)) + 16 + static_cast<int>(sizeof(mk::GemvShared)) + 16 +
           stages * static_cast<int>(sizeof(MkChunk)) + 8 * (nphases + 1);
}

int mk_max_stages(int x_bytes, int rec_chunks, int batch, int d_head, int nphases) {
    const int budget = 227 * 1024 - 1024;  // dynamic shared memory per CTA (+ static / alignment slack)
    int s = (budget - mk_smem_bytes(0, x_bytes, rec_chunks, batch, d_head, nphases)) / kChunkBytes;
    while (s > 0 && mk_smem_bytes(s, x_bytes, rec_chunks, batch, d_head, nphases) > budget) --s;
    return s;
}

int mk_consumer_warps() { return mk::kConsumerWarps; }

namespace {
template <typename W, int B, int DH>
int max_pairs_t(int smem_bytes) {
    auto fn = mk::decode_mk_kernel<W, B, DH>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(mk::kThreads);
    cfg.dynamicSmemBytes = smem_bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}
}  // namespace

int mk_max_active_pairs(WType wt, int batch, int d_head, int smem_bytes) {
#define FSVD_MKP(W, BB, DHH) \
    if (batch == BB && d_head == DHH) return max_pairs_t<W, BB, DHH>(smem_bytes);
    if (wt == kBF16) {
        FSVD_MKP(__nv_bfloat16, 1, 128) FSVD_MKP(__nv_bfloat16, 2, 128) FSVD_MKP(__nv_bfloat16, 1, 64)
        FSVD_MKP(__nv_bfloat16, 2, 64) FSVD_MKP(__nv_bfloat16, 1, 32) FSVD_MKP(__nv_bfloat16, 2, 32)
    } else {
        FSVD_MKP(float, 1, 128) FSVD_MKP(float, 2, 128) FSVD_MKP(float, 1, 64) FSVD_MKP(float, 2, 64)
        FSVD_MKP(float, 1, 32) FSVD_MKP(float, 2, 32)
    }
#undef FSVD_MKP
    return 0;
}

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
