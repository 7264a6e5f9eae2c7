// Device scan + stable LSD radix sort used by tile binning.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace nx {

void count_launch(int n);

constexpr int kScanItems = 4;        // per thread
constexpr int kScanThreads = 1024;
constexpr int kScanTile = kScanItems * kScanThreads;
constexpr int64_t kScanLoopMax = 16 * kScanTile;  // single-launch scan up to 64K values
constexpr int kRadixThreads = 256;
#ifndef NX_RADIX_TILE
#define NX_RADIX_TILE 2048
#endif
constexpr int kRadixTile = NX_RADIX_TILE;  // items per block per pass (look-back chains of n / tile blocks)
// 64-bit (depth) sorts: ~180K keys at config 2, latency-bound; the tile is a separate
// knob (smaller tiles = more blocks and shorter ranking chains, measured no faster)
#ifndef NX_RADIX_TILE64
#define NX_RADIX_TILE64 2048  // measured at config 2: 2048 473.3, 1024 471.2, 512 469.7, 256 462.8 frames/s
// (again with the batched look-back: 2048 488.5, 1024 485.3, 512 479.7; 32-bit tile
// 4096 489.1, 1024 482.4; look-back batch 16 483.6 vs 8)
#endif
constexpr int kRadixTile64 = NX_RADIX_TILE64;
constexpr int kRadixBits = 8;
constexpr int kRadixBuckets = 1 << kRadixBits;

// Exclusive prefix sum of n int32 values (n <= kScanTile^2). out may alias in.
// If total != nullptr the grand total is stored there (device).
// Scratch: scan_scratch_ints(n) ints.
size_t scan_scratch_ints(int64_t n);
void scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int32_t* total, int32_t* scratch,
                    cudaStream_t stream);

// Stable LSD radix sort of (key, value) pairs over key bits [begin_bit, end_bit).
// Ping-pongs between (keys, vals) and (keys_alt, vals_alt); returns true if the
// sorted result ended in the *_alt buffers. Scratch: radix_scratch_ints(n) ints.
// n is the host-side capacity (grid size); if n_dev != nullptr the actual count is
// read on the device (no host round trip), capped by n.
size_t radix_scratch_ints(int64_t n);    // for radix_sort_pairs_u32
size_t radix_scratch_ints64(int64_t n);  // for radix_sort_pairs_u64
bool radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                          int64_t n, const int32_t* n_dev, int begin_bit, int end_bit, int32_t* scratch,
                          cudaStream_t stream);
bool radix_sort_pairs_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                          int64_t n, const int32_t* n_dev, int begin_bit, int end_bit, int32_t* scratch,
                          cudaStream_t stream);

}  // namespace nx
