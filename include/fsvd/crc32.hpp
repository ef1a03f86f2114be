#pragma once
// CRC-32/IEEE (reflected 0xEDB88320), as used by the FSVD15 per-tensor
// checksums (reference proj/include/fsvd/crc32.hpp:10-34). Slice-by-8 table
// walk: same polynomial and result, ~8x the reference's byte-wise speed,
// which matters when validating a 15 GB LLaMA-7B-shape checkpoint.

#include <cstddef>
#include <cstdint>
#include <cstring>

namespace fsvd {

namespace detail {
struct Crc32Tables {
    uint32_t t[8][256];
    constexpr Crc32Tables() : t{} {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? 0xEDB88320u : 0u);
            t[0][i] = c;
        }
        for (uint32_t i = 0; i < 256; ++i)
            for (int s = 1; s < 8; ++s) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xFFu];
    }
};
inline constexpr Crc32Tables kCrc32Tables{};
}  // namespace detail

inline uint32_t crc32_update(uint32_t crc, const void* bytes, size_t len) {
    const auto& T = detail::kCrc32Tables.t;
    const auto* p = static_cast<const unsigned char*>(bytes);
    crc = ~crc;
    while (len >= 8) {
        uint32_t lo, hi;
        std::memcpy(&lo, p, 4);
        std::memcpy(&hi, p + 4, 4);
        lo ^= crc;
        crc = T[7][lo & 0xFF] ^ T[6][(lo >> 8) & 0xFF] ^ T[5][(lo >> 16) & 0xFF] ^ T[4][lo >> 24] ^
              T[3][hi & 0xFF] ^ T[2][(hi >> 8) & 0xFF] ^ T[1][(hi >> 16) & 0xFF] ^ T[0][hi >> 24];
        p += 8;
        len -= 8;
    }
    while (len--) crc = T[0][(crc ^ *p++) & 0xFFu] ^ (crc >> 8);
    return ~crc;
}

inline uint32_t crc32(const void* bytes, size_t len) { return crc32_update(0u, bytes, len); }

}  // namespace fsvd
