// sort.cuh -- device-wide stable LSD radix sort of (uint64 key, uint32 value)
// pairs, 8-bit digits: per pass a digit histogram per tile, one scan over
// (digit, tile), and a stable scatter (match_any ranks within a warp, warp
// prefixes within a tile).  Used by the text readers (id densification,
// the METIS symmetry check).
#pragma once

#include "common.cuh"

namespace cdk {

// Sorts keys[0, n) (and vals alongside, if non-null) by bits [0, end_bit).
void radix_sort_pairs(cd_ctx *ctx, uint64_t *keys, uint32_t *vals, int64_t n, int end_bit);

}  // namespace cdk
