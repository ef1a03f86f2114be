// Phase program of the persistent decode megakernel (decode_mk.cu).
//
// A decode step is a list of phases separated by grid barriers. Each CTA has
// one producer warp that streams the weight tiles of every GEMV phase of the
// launch, in order, through a shared-memory ring (cp.async.bulk), never
// waiting for activations; the consumer warps stage a phase's input vector
// (one bulk copy of a ready-made "planes" buffer), reduce the ring's chunks
// on the tensor cores, and finalize the phase's outputs.
//
// Output exchange: a CTA owns a contiguous range of (16-row tile, 128-byte
// line) units. An output tile covered by one CTA is finalized by that CTA; a
// tile shared by several CTAs is finalized by the last of them to arrive (a
// per-tile counter), which sums the per-CTA partials ("pieces") in CTA order
// -- deterministic bits for any launch structure (eager / per layer / full
// step are bitwise identical). Finalizing applies the epilogue
// once per row: RoPE + KV append, residual add + next RMSNorm's gamma,
// SiLU.mul, logits, and writes the next phase's input planes.
#pragma once

#include <vector>

#include "kernels.h"

namespace fsvd::k {

enum MkKind : int { kMkGemv = 0, kMkAttn = 1, kMkArgmax = 2, kMkVec = 3 };

// An activation vector in the form the GEMV consumes as its B operand:
// bf16 weights: [B][2][len] bf16 (x = hi + lo, both RNE: fp32-grade
// activations on bf16 tensor cores); fp32 weights: [B][len] fp32.
// len is a multiple of 64 elements, padding stays zero.
struct Planes {
    void* p;
    int len;
};

enum MkOut : int {
    kOutPlanes = 0,  // out.p[x_off[s] + r] = v                       (rank spaces)
    kOutResid = 1,   // xres[r] += v; out = xres[r] * gamma[r]         (o / down B)
    kOutQKV = 2,     // q: RoPE -> qbuf; k: RoPE -> K cache[pos]; v -> V cache[pos]
    kOutSilu = 3,    // dual: out = silu(gate) * up                     (up/gate B)
    kOutLogits = 4,  // logits[b][r] = v, per-tile best -> cand        (head)
};

struct MkGemv {
    GemvSeg seg[3];   // weights; seg.x_off = the segment's offset in the input planes
    int nseg;
    int dual;         // seg0 = up, seg1 = gate: per tile, up lines then gate lines
    int exact_split;  // even unit split over the CTAs; tiles shared by CTAs go through the pieces exchange
    Planes in;
    const float* norm_src;  // non-null: output *= inv_rms(norm_src[b][0..norm_len)) (RMSNorm)
    int norm_ld, norm_len;
    float eps;
    int out_kind;
    Planes out;
    int out_off[3];   // kOutPlanes: output offset of each segment's rows
    float* xres;      // kOutResid: fp32 residual [B][xres_ld]
    int xres_ld;
    const float* gamma;  // kOutResid: the next RMSNorm's gamma
    // kOutQKV
    float* qbuf;      // [B][q_ld] RoPE'd q
    int q_ld;
    const float2* rope;  // [cap][d_head/2] (cos, sin), angles in double on the host
    void* kcache;
    void* vcache;
    long long cache_bstride, cache_hstride;
    int d_head;
    const int* pos;
    int attn_pairs;   // the attention that follows runs one CTA pair per (b, h) (MkAttn::pairs)
    // kOutLogits
    float* logits;    // [B][vocab]
    int vocab;
    float* cand_v;    // [tiles][B] best logit of each 16-row tile (ties -> lowest index)
    int* cand_i;
    // pieces exchange (per phase)
    float* pieces;    // [out tile][max_pieces][subs][16][B]
    unsigned* count;  // [out tile], zero between uses (self-resetting)
    int max_pieces;
    // chunk records in shared memory: [local tile < rec_ntl][sub][c < rec_c[sub]][16][B]
    int rec_ntl, rec_c0, rec_c1;
};

struct MkAttn {
    const float* qbuf;  // [B][q_ld] RoPE'd q of the current position
    int q_ld;
    const void* kcache;  // layer base [B][H][cap][d_head]
    const void* vcache;
    long long cache_bstride, cache_hstride;
    const int* pos;      // attend rows 0 .. *pos
    float* partial;      // [B*H][splits][d_head + 2]: acc, l, m
    unsigned* count;     // [B*H]
    int n_heads, d_head, splits;
    float scale;
    Planes out;          // merged output (o-projection input)
    int pairs;           // 1: one CTA pair (a cluster of 2) per (b, h), halves merged through DSMEM
};

struct MkArgmax {
    const float* cand_v;  // head tile candidates
    const int* cand_i;
    int ntiles;
    int* tokens;          // [B] next input token
    int* pos;             // length register
    int pos_inc;
    int* out;             // generated tokens [B][out_ld] at column *step (may be null)
    int out_ld;
    int* step;
};

struct MkVec {
    const void* emb;     // embedding [V][emb_ld] (weight dtype), rows tokens[b]; or null
    int emb_ld;
    const int* tokens;
    const float* src;    // else: fp32 [B][src_ld]
    int src_ld;
    int len;
    float* xres;         // optional copy of the vector (the residual stream)
    int xres_ld;
    const float* gamma;  // planes = x * gamma
    Planes out;
};

struct alignas(16) MkPhase {
    int kind;
    MkGemv g;
    MkAttn a;
    MkArgmax m;
    MkVec v;
};

// One ring chunk of a CTA's weight stream, precomputed on the host (the
// producer and the consumers never walk the work split on the device).
struct alignas(16) MkChunk {
    const char* src;   // weights, <= kChunkLines contiguous 2 KiB line tiles
    uint16_t T;        // output tile
    uint16_t kbase;    // input element offset of the chunk's first line
    uint8_t nl;        // lines | 0x10: gate half (sub 1) | 0x20: last chunk of its output tile
    uint8_t k;         // output tile index local to the CTA's range (chunk records)
    uint8_t c;         // chunk index inside its run (record slot)
    uint8_t ctile;     // chunk index inside its output tile
};

struct MkLaunch {
    const MkPhase* phases;  // device array
    int p_begin, p_end;
    int reps;               // >= 1: run phases [p_begin, p_end) reps times (multi-step decode launch)
    unsigned* bar;          // zero-initialized grid-barrier counter (self-resetting)
    int grid, smem_bytes;
    int stages;             // ring depth (kChunkBytes each)
    int x_bytes;            // staged input region
    int rec_chunks;         // per-phase chunk records
    int l2_ahead;           // weight chunks prefetched into L2 beyond the ring
    const int* pos;         // length register (constant during a launch but for the final argmax phase)
    const MkChunk* chunks;  // [cta][...] chunk records of every phase
    const int* chunk_start; // [cta][nphases + 1] first record of each phase
    const int* chunk_tiles; // [cta][nphases] first | last output tile << 16 of the CTA's range (-1: none)
    int nphases;
    volatile int* progress; // optional host-mapped [grid][16] for hang diagnosis
    unsigned long long* trace;  // optional [grid][phases][4] %globaltimer stamps
    int cluster2;               // launch as clusters of 2 CTAs (the attention pairs)
};

#ifndef FSVD_MK_CHUNK_LINES
#define FSVD_MK_CHUNK_LINES 11  // swept 4-15 on B200: 11 lines x 7 stages is the best trade of per-chunk cost vs ring depth
#endif
constexpr int kChunkLines = FSVD_MK_CHUNK_LINES;          // ring chunk: <= kChunkLines lines of one tile (<= 15: 4-bit field)
constexpr int kChunkBytes = kChunkLines * kLineTileBytes;  // 22 KiB
constexpr int kMkMaxStages = 32;                           // ring slots (bounded by shared memory)

// ---- host mirrors of the device work split ----
// Units (16-row x 128-byte lines) of a GEMV phase.
int mk_units(const GemvSeg* seg, int nseg, int dual, int esize);
// Output tiles (dual: up/gate tile pairs count once).
int mk_out_tiles(const GemvSeg* seg, int nseg, int dual, int esize);
// Max CTAs contributing to one output tile; chunk-record shape of a CTA
// (max local tiles, max chunks per run for sub 0 / 1).
void mk_split_stats(const GemvSeg* seg, int nseg, int dual, int esize, int grid, int exact, int* max_pieces,
                    int* rec_ntl, int* rec_c0, int* rec_c1);
constexpr int kMkMaxLocalTiles = 64;
// Chunk records of every GEMV phase for a grid of `grid` CTAs.
void mk_build_chunks(const struct MkPhase* phases, int nphases, int grid, int esize, std::vector<MkChunk>& out,
                     std::vector<int>& start, std::vector<int>& tiles);
int mk_smem_bytes(int stages, int x_bytes, int rec_chunks, int batch, int d_head, int nphases);
int mk_max_stages(int x_bytes, int rec_chunks, int batch, int d_head, int nphases);
int mk_consumer_warps();
// false if (wt, batch, d_head) has no instantiation
// co-resident 2-CTA clusters of the megakernel at the given shared memory (0 if unknown)
int mk_max_active_pairs(WType wt, int batch, int d_head, int smem_bytes);
bool mk_launch(WType wt, int batch, int d_head, const MkLaunch& L, cudaStream_t s);

}  // namespace fsvd::k
