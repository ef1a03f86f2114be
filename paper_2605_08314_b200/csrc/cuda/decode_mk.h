// Phase program of the persistent decode megakernel (decode_mk.cu).
//
// Only the grid barrier synchronizes CTAs: a GEMV phase writes per-CTA
// partial sums ("pieces") of its output rows, and the consuming phase's
// input staging sums the pieces in CTA order and applies the producer's
// epilogue (residual add, SiLU.mul, RoPE + KV append, attention merge).
#pragma once

#include "kernels.h"

namespace fsvd::k {

enum MkKind : int { kMkGemv = 0, kMkAttn = 1, kMkArgmax = 2 };

// Pieces of a producer phase, slot-plane major: output row r (segment tiles
// concatenated, 16 rows each), CTA slot j < S, batch b at base[(j*R + r)*B + b].
// Every phase owns its buffer and a tile's unused slots stay zero (never
// written), so a consumer sums all S planes without knowing the piece count.
struct Pieces {
    float* base;
    int R;  // rows (output tiles * 16)
    int S;  // slots (max pieces on any tile)
};

// One output segment of a producer, as seen by a consumer's input vector:
// x[x_off + r] for r < rows comes from tile tbase + r/16, row r%16 of pc.
struct InSeg {
    int x_off, rows, tbase;
    Pieces pc;
};

enum InKind : int {
    kInPlain = 0,     // x = src
    kInPieces = 1,    // x = sum(pieces) over the segments
    kInResidual = 2,  // x = src + sum(pieces of seg[0]) (nseg 0: x = src); written back to dst
    kInSilu = 3,      // x[r] = silu(sum gate) * sum(up), up = seg[0], gate = seg[1]
    kInAttn = 4,      // x = merged attention partials (all heads)
    kInEmbed = 5,     // x = E[tokens[b]] (weight dtype); written back to dst
};

struct AttnMerge {
    const float* partial;  // [B*H][splits][d_head + 4] (acc, l, m)
    int n_heads, d_head, splits;
    const int* pos;        // attended positions 0 .. *pos
};

struct InputSpec {
    int kind;
    const float* src;  // [B][src_ld]
    int src_ld;
    float* dst;        // kInResidual write-back [B][dst_ld] (each CTA writes its slice)
    int dst_ld;
    int len;           // logical length of src/dst (kInResidual, kInPlain, kInEmbed)
    const void* emb;   // kInEmbed: [V][emb_ld] weight dtype
    int emb_ld;
    const int* tokens; // kInEmbed: [B]
    InSeg seg[3];
    int nseg;
    AttnMerge am;
};

struct MkGemv {
    GemvSeg seg[3];      // weights (epi unused: the consumer applies it)
    int nseg;
    int dual;            // seg0 = up, seg1 = gate: units interleaved per tile
    InputSpec in;
    int x_len;           // staged elements per batch row (>= every seg's x_off + kp)
    const float* gamma;  // RMSNorm if non-null
    float eps;
    int norm_len;
    Pieces out;          // this phase's pieces
};

struct MkAttn {
    // q/k/v for the current position from the QKV-reconstruction pieces
    Pieces pc;
    int tbase_q, tbase_k, tbase_v;  // tiles of the q/k/v segments (each d_model rows)
    const float2* rope;             // [cap][d_head/2]
    const void* kcache;             // layer base [B][H][cap][d_head]
    const void* vcache;
    long long cache_bstride, cache_hstride;
    const int* pos;
    float* partial;                 // [B*H][splits][d_head + 4]: acc, l, m
    int n_heads, d_head, splits;
    float scale;
    float* q_out;                   // optional debug copy of RoPE'd q [B][d] (nullptr: none)
};

struct MkArgmax {
    Pieces pc;          // head pieces (one segment, tbase 0)
    int vocab;
    float* logits;      // [B][vocab]
    float* best_v;      // [grid][B]
    int* best_i;
    unsigned* ticket;   // zeroed, self-resetting
    int* tokens;        // [B] next input token
    int* pos;           // length register
    int pos_inc;
    int* out;           // generated tokens [B][out_ld] at column *step (may be null)
    int out_ld;
    int* step;
};

struct MkPhase {
    int kind;
    MkGemv g;
    MkAttn a;
    MkArgmax m;
};

struct MkLaunch {
    const MkPhase* phases;  // device array
    int p_begin, p_end;
    unsigned* bar;          // zero-initialized grid-barrier counter (self-resetting)
    int region_bytes;       // shared region carved per phase: x planes + unit partials
    int red_floats;         // scratch: attention warp states / per-head merge records
    int grid, smem_bytes;
    unsigned long long* trace;  // optional [grid][phases][8] globaltimer stamps (profiling)
};

// Output tiles of a GEMV phase (dual: up tiles then gate tiles).
int mk_out_tiles(const GemvSeg* seg, int nseg, int dual, int esize);
// Host mirror of the device unit split: fills npieces[T] for every output
// tile of a GEMV phase; returns the max (the phase's piece stride S).
int mk_npieces(const GemvSeg* seg, int nseg, int dual, int esize, int grid, uint8_t* npieces);
// Units of a GEMV phase (all segments).
int mk_units(const GemvSeg* seg, int nseg, int dual, int esize);
int mk_region_bytes(int batch, WType wt, int x_len, int units_per_cta);
int mk_red_floats(int batch, int n_heads, int d_head);
int mk_smem_bytes(int region_bytes, int red_floats);
int mk_warps();
// false if (wt, batch, d_head) has no instantiation
bool mk_launch(WType wt, int batch, int d_head, const MkLaunch& L, cudaStream_t s);

}  // namespace fsvd::k
