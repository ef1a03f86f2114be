// Device weight layout shared by the decode megakernel and the prefill GEMMs.
//
// Every factor matrix is stored transposed (output-major: row n = output n,
// K = reduction dim) in 16-row tiles. A tile is a sequence of 128-byte
// "lines" along K: line l holds 128 bytes of each of the 16 rows (2 KiB),
// row i at byte 128*i, and inside row i the 16-byte chunks are XOR-swizzled
// by (i & 7). This is exactly the K-major SWIZZLE_128B core-matrix layout of
// the tcgen05 UMMA descriptors (8-row x 128-byte atoms), so prefill TMA-loads
// it verbatim, and it makes the decode tensor-core GEMV's shared-memory reads
// bank-conflict-free. Decode streams a tile in "units" of kUnitLines lines
// (8 KiB), one contiguous cp.async.bulk each.
//
// K is zero-padded to a whole line (64 bf16 / 32 fp32 elements); rows are
// zero-padded to a whole tile. Padding contributes exactly 0.
#pragma once

#include <stddef.h>
#include <stdint.h>

#ifndef __CUDACC__
#define FSVD_HD inline
#else
#define FSVD_HD __host__ __device__ __forceinline__
#endif

namespace fsvd::k {

constexpr int kLineBytes = 128;
constexpr int kTileRows = 16;
constexpr int kLineTileBytes = kLineBytes * kTileRows;  // 2 KiB
constexpr int kUnitLines = 4;
constexpr int kUnitBytes = kLineTileBytes * kUnitLines;  // 8 KiB

struct WLayout {
    int rows;   // logical rows (outputs)
    int k;      // logical K
    int kp;     // padded K (multiple of line elements)
    int esize;  // 2 (bf16) or 4 (fp32)

    FSVD_HD int line_elems() const { return kLineBytes / esize; }
    FSVD_HD int nlines() const { return kp / line_elems(); }
    FSVD_HD int ntiles() const { return (rows + kTileRows - 1) / kTileRows; }
    FSVD_HD int nunits() const { return (nlines() + kUnitLines - 1) / kUnitLines; }
    FSVD_HD size_t tile_bytes() const { return static_cast<size_t>(nlines()) * kLineTileBytes; }
    FSVD_HD size_t bytes() const { return static_cast<size_t>(ntiles()) * tile_bytes(); }
    // byte offset of element (r, kk)
    FSVD_HD size_t offset(int r, int kk) const {
        const int tile = r >> 4, i = r & 15, le = line_elems();
        const int line = kk / le, within = kk - line * le;
        const int byte = within * esize;
        return static_cast<size_t>(tile) * tile_bytes() + static_cast<size_t>(line) * kLineTileBytes + i * kLineBytes +
               ((((byte >> 4) ^ (i & 7)) << 4) | (byte & 15));
    }
};

FSVD_HD int pad_line(int k, int esize) {
    const int le = kLineBytes / esize;
    return (k + le - 1) / le * le;
}

FSVD_HD WLayout make_layout(int rows, int k, int esize) { return WLayout{rows, k, pad_line(k, esize), esize}; }

}  // namespace fsvd::k
